# strip-length A/B for the telescoped 2D+2V stage kernel: every setting REPS times, interleaved
cd $GRAFT_REPO_ROOT
O=gpurun_out/strips; mkdir -p $O
: > $O/exp.log
for rep in 1 2 3; do
for cfg in ${CFGS:-1 "52,12" "49,15" "54,10" "56,8" "50,14" "60,4"}; do
  export VLASOV_STRIPS2T="$cfg"
  timeout 300 python bench.py --workload C5 --steps 30 --no-cpu-baseline > $O/b5.json 2> $O/b5.err
  python -c "
import json; d=json.load(open('$O/b5.json')); print('$cfg', round(d['value']/1e9,2), round(d['ms_per_step'],4), [round(x*1e3,1) for x in d['roofline']['stage_ms_eager']], d['clocks']['sm_mhz'])" >> $O/exp.log 2>&1
done
done
sort $O/exp.log

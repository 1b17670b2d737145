# build-flag experiments for the 1D+1V stage kernel (each config: rebuild on the box, C4 bench twice)
cd $GRAFT_REPO_ROOT
O=gpurun_out/cfg; mkdir -p $O; : > $O/exp.log
for cfg in "$@"; do
  VLASOV_NVCC_FLAGS="$cfg" python -c "from paper_1204_3853_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  for rep in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('cfg [$cfg]', round(d['value']/1e9,2), round(d['ms_per_step'],4), [round(x*1e3,1) for x in d['roofline']['stage_ms_eager']])" >> $O/exp.log 2>&1
  done
done
cat $O/exp.log

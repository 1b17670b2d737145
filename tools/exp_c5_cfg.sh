# build-flag experiments for the 2D+2V stage kernel (each config: rebuild, C5 bench)
cd $GRAFT_REPO_ROOT
for cfg in "$@"; do
  VLASOV_NVCC_FLAGS="$cfg" python -c "from paper_1204_3853_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== $cfg" >> gpurun_out/exp5.log
  python bench.py --workload C5 --steps 10 --no-cpu-baseline > gpurun_out/exp_b5.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/exp_b5.json')); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'], [round(x*1e3,1) for x in d['roofline']['stage_ms']])" >> gpurun_out/exp5.log 2>&1
done

# strip-shift experiments: which stages start their strips half a strip later (VLASOV_XSHIFT_MASK)
cd $GRAFT_REPO_ROOT
O=gpurun_out/xshift; mkdir -p $O; : > $O/exp.log
for rep in 1 2; do
for m in 0x14 0x1c 0x04 0x0c 0x00 0x10 0x18; do
  VLASOV_XSHIFT_MASK=$m timeout 300 python bench.py --steps 20 --no-cpu-baseline > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('mask', '$m', round(d['value']/1e9,2), round(d['ms_per_step'],4), [round(v*1e3,1) for v in d['roofline']['stage_ms_eager']])" >> $O/exp.log 2>&1
done; done
sort $O/exp.log

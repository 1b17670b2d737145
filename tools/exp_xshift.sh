cd $GRAFT_REPO_ROOT
O=gpurun_out/xshift; mkdir -p $O; : > $O/exp.log
for rep in 1 2; do
for x in 2 0 1 3; do
  VLASOV_XSHIFT=$x timeout 300 python bench.py --steps 20 --no-cpu-baseline > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('xshift', $x, round(d['value']/1e9,2), round(d['ms_per_step'],4), [round(v*1e3,1) for v in d['roofline']['stage_ms_eager']])" >> $O/exp.log 2>&1
done; done
sort $O/exp.log

cd $GRAFT_REPO_ROOT
O=gpurun_out/gsteps; mkdir -p $O; : > $O/exp.log
for rep in 1 2; do
for wl in C4 C5; do
for g in 1 2 5 10 20; do
  timeout 300 python bench.py --workload $wl --steps 20 --graph-steps $g --no-cpu-baseline > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('$wl', $g, round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['roofline']['frac'],3))" >> $O/exp.log 2>&1
done; done; done
sort $O/exp.log

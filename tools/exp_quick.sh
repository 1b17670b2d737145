cd $GRAFT_REPO_ROOT
O=gpurun_out/fin; mkdir -p $O
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --workload C5 --steps 10 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --workload C5P --steps 10 --no-cpu-baseline > $O/bench_c5p.json 2> $O/bench_c5p.err
timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "bench or smoke or c1_one_step" > $O/pytest_small.txt 2>&1
tail -2 $O/pytest_small.txt
python -c "
import json
for n in ('c4','c5','c5p'):
    d=json.load(open('$O/bench_%s.json'%n)); print(n, round(d['value']/1e9,2), d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], (d.get('cpu_baseline') or {}).get('value'))
"

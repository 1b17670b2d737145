cd $GRAFT_REPO_ROOT
O=gpurun_out/quick; mkdir -p $O; : > $O/exp.log
timeout 900 python -m pytest tests/test_gpu_uniform.py tests/test_gpu_vslab.py -m gpu -x -q -p no:cacheprovider > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt >> $O/exp.log
for rep in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print(round(d['value']/1e9,2), round(d['ms_per_step'],4), d['roofline']['frac'], [round(x*1e3,1) for x in d['roofline']['stage_ms_eager']])" >> $O/exp.log 2>&1
done
cat $O/exp.log

cd $GRAFT_REPO_ROOT
O=gpurun_out/split; mkdir -p $O; : > $O/exp.log
timeout 900 python -m pytest tests/test_gpu_uniform.py -m gpu -x -q -p no:cacheprovider -k "split" > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt >> $O/exp.log
VLASOV_FIELD=split timeout 900 python -m pytest tests/test_gpu_uniform.py tests/test_gpu_physics.py tests/test_gpu_vslab.py -m gpu -x -q -p no:cacheprovider > $O/pytest_split_env.txt 2>&1
tail -3 $O/pytest_split_env.txt >> $O/exp.log
for rep in 1 2 3; do
for x in toeplitz split; do
  VLASOV_FIELD=$x timeout 300 python bench.py --steps 20 --no-cpu-baseline > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('field', '$x', round(d['value']/1e9,2), round(d['ms_per_step'],4), [round(v*1e3,1) for v in d['roofline']['stage_ms_eager']])" >> $O/exp.log 2>&1
done; done
cat $O/exp.log

cd $GRAFT_REPO_ROOT
O=gpurun_out/split_ab; mkdir -p $O; : > $O/exp.log
for rep in 1 2; do
for lib in new old; do
  cp libs_ab/lib_$lib.so paper_1204_3853_b200/libvlasov.so; touch paper_1204_3853_b200/libvlasov.so
  for x in toeplitz split; do
  VLASOV_FIELD=$x timeout 300 python bench.py --steps 20 --no-cpu-baseline > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('lib', '$lib', 'field', '$x', round(d['value']/1e9,2), round(d['ms_per_step'],4), [round(v*1e3,1) for v in d['roofline']['stage_ms_eager']])" >> $O/exp.log 2>&1
  done
done; done
cat $O/exp.log
cp libs_ab/lib_old.so paper_1204_3853_b200/libvlasov.so; touch paper_1204_3853_b200/libvlasov.so
VLASOV_FIELD=split timeout 900 python -m pytest tests/test_gpu_uniform.py -m gpu -x -q -p no:cacheprovider -k "strip_shift or split or deterministic or c2_hundred or c1" > $O/pytest_t3.txt 2>&1
tail -3 $O/pytest_t3.txt

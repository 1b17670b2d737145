cd $GRAFT_REPO_ROOT
O=gpurun_out/l2hint; mkdir -p $O; : > $O/exp.log
timeout 900 python -m pytest tests/test_gpu_uniform.py -m gpu -x -q -p no:cacheprovider -k "c1 or c2_hundred or deterministic or c4_full_size_one" > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt >> $O/exp.log
for rep in 1 2; do
for x in 1 0; do
  VLASOV_L2HINT=$x timeout 300 python bench.py --steps 20 --no-cpu-baseline > $O/b.json 2> $O/b.err
  python -c "
import json; d=json.load(open('$O/b.json')); print('l2hint', $x, round(d['value']/1e9,2), round(d['ms_per_step'],4), [round(v*1e3,1) for v in d['roofline']['stage_ms_eager']])" >> $O/exp.log 2>&1
done; done
PS="python tools/profile_step.py --steps 3"
for x in 1 0; do
VLASOV_L2HINT=$x timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none --cache-control none -k regex:k_stage_1d1v -c 12 --csv --log-file $O/launches_hint$x.csv $PS > $O/ncu_$x.log 2>&1
done
cat $O/exp.log

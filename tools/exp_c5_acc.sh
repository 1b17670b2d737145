# accumulator-form 2D+2V stage kernel: tests, C5 bench per strip setting, ncu launch list + full capture
cd $GRAFT_REPO_ROOT
O=gpurun_out/acc; mkdir -p $O
: > $O/exp.log
timeout 900 python -m pytest tests/test_gpu_2d2v.py tests/test_gpu_n3.py -m gpu -x -q -p no:cacheprovider > $O/pytest.txt 2>&1
tail -15 $O/pytest.txt >> $O/exp.log
for cfg in ${CFGS:-auto 1 2 "52,12"}; do
  echo "== $cfg" >> $O/exp.log
  if [ "$cfg" = auto ]; then unset VLASOV_STRIPS2A; else export VLASOV_STRIPS2A="$cfg"; fi
  timeout 300 python bench.py --workload C5 --steps 20 --no-cpu-baseline > $O/b5.json 2> $O/b5.err
  python -c "
import json; d=json.load(open('$O/b5.json')); print(d['value']/1e9, d['ms_per_step'], d['roofline']['frac'], [round(x*1e3,1) for x in d['roofline']['stage_ms_eager']])" >> $O/exp.log 2>&1
  tail -2 $O/b5.err >> $O/exp.log
done
unset VLASOV_STRIPS2A
if [ -n "$NCU" ]; then
P5="python tools/profile_step.py --workload C5 --steps 2"
timeout 300 $P5 > $O/plain5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none -c 100 --csv --log-file $O/launches_c5.csv $P5 > $O/ncu_launch_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_2d2v -s 4 -c 4 -o $O/full_c5 $P5 > $O/ncu_full_c5.log 2>&1
fi
cat $O/exp.log

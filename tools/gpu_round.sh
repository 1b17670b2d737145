#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list and one full capture of the stage kernel.
# usage: TAG=name [SKIP_TESTS=1] [NCU_FULL=regex] bash tools/gpu_round.sh
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${TAG:-run}
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
timeout 600 python bench.py ${BENCH_ARGS} > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
PS="python tools/profile_step.py --steps 3 ${PROF_ARGS}"
timeout 300 $PS > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
   --log-file $O/launches.csv $PS > $O/ncu_launch.log 2>&1
if [ -n "$NCU_FULL" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$NCU_FULL -s 8 -c 4 \
   -o $O/full $PS > $O/ncu_full.log 2>&1
fi
ls -la $O

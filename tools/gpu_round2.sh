#!/bin/bash
# Round-2 measured artefacts: full GPU test suite, smoke, bench lines (C4 headline with the CPU
# baseline, C5, C5P, C3 with its CPU baseline, v-slab N=1, reference arm), regrid phase times,
# ncu launch lists (C4, C5) and full captures of the stage kernels (the 4 launches of one step,
# with the L2 write-sector metric for tools/traffic_from_ncu.py).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${TAG:-r2}
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
fi
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --workload C5 --steps 10 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --workload C5P --steps 10 --no-cpu-baseline > $O/bench_c5p.json 2> $O/bench_c5p.err
timeout 900 python bench.py --workload C3 --steps 20 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --shard vslab --steps 10 --no-cpu-baseline > $O/bench_vslab1.json 2> $O/bench_vslab1.err
VLASOV_VSLAB_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --shard vslab --steps 10 --no-cpu-baseline > $O/bench_vslab1_nccl.json 2> $O/bench_vslab1_nccl.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 python tools/time_regrid.py > $O/regrid_phases.txt 2>&1
PS="python tools/profile_step.py --steps 3"
timeout 300 $PS > $O/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none -c 200 --csv \
   --log-file $O/launches_c4.csv $PS > $O/ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_1d1v -s 8 -c 4 \
   -o $O/full_c4 $PS > $O/ncu_full_c4.log 2>&1
P5="python tools/profile_step.py --workload C5 --steps 2"
timeout 300 $P5 > $O/plain5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none -c 100 --csv \
   --log-file $O/launches_c5.csv $P5 > $O/ncu_launch_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_2d2v -s 4 -c 4 \
   -o $O/full_c5 $P5 > $O/ncu_full_c5.log 2>&1
ls -la $O

cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/r2c; mkdir -p $O
P5="python tools/profile_step.py --workload C5 --steps 2"
timeout 300 $P5 > $O/plain5.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 100 --csv --log-file $O/launches_c5.csv $P5 > $O/ncu_launch_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_2d2v_tel -s 4 -c 4 -o $O/full_c5 $P5 > $O/ncu_full_c5.log 2>&1
ls -la $O

# full GPU suite, smoke, then the C4 / C5 / C5P bench lines (quick check of a change)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out/${TAG:-chk}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -5 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --workload C5 --steps 20 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --workload C5P --steps 20 --no-cpu-baseline > $O/bench_c5p.json 2> $O/bench_c5p.err
python - <<PY
import json
for n in ("c4","c5","c5p"):
    try:
        d=json.load(open("$O/bench_%s.json"%n)); print(n, round(d["value"]/1e9,2), round(d["ms_per_step"],4), round(d["roofline"]["frac"],3), [round(x*1e3,1) for x in d["roofline"].get("stage_ms_eager",[])])
    except Exception as e: print(n, "failed", e)
PY

# build-flag experiments with the stage-kernel phase trace (each config: rebuild with
# -DSTAGE1D_TRACE plus the flags, run tools/trace_stage.py)
cd $GRAFT_REPO_ROOT
for cfg in "$@"; do
  VLASOV_NVCC_FLAGS="-DSTAGE1D_TRACE $cfg" python -c "from paper_1204_3853_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== $cfg"
  python tools/trace_stage.py C4 2>&1 | grep -E "fused=True|end by vtile"
done

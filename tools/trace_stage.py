"""Phase timeline of the 1D+1V stage kernel (build with VLASOV_NVCC_FLAGS=-DSTAGE1D_TRACE): per-CTA
%globaltimer stamps -> percentiles (us after the first CTA started) of: 0 start, 1 after the
cluster barrier, 2 rho (+gE) landed, 3 mean, 4 own E rows done, 5 E of the tile ready, 6 first ring
slot consumed, 7 end."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1204_3853_b200 import _lib  # noqa: E402
from paper_1204_3853_b200.solver import UniformVlasov1D  # noqa: E402

w = inputs.get(sys.argv[1] if len(sys.argv) > 1 else "C4")
dt = inputs.fixed_dt(w)
fn = _lib.lib.vlasov_debug_stage_trace
fn.argtypes = [C.c_void_p, C.c_int]
for fused in (True, False):
    S = UniformVlasov1D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w), inputs.background_profile(w),
                        fused=fused)
    S.set_state(inputs.initial_cell_averages(w))
    for _ in range(3):
        S.step(dt)
    nb = 2048
    for s in (1, 2, 3, 4):
        buf = np.zeros((nb, 10), dtype=np.uint64)
        fn(buf.ctypes.data, nb)              # clear is not needed: rows of this launch overwrite
        with torch.cuda.stream(S.stream):
            S.field_launch(s)
            S.stream.synchronize()
            S.stage_launch(s, dt)
        S.stream.synchronize()
        fn(buf.ctypes.data, nb)
        n = int((buf[:, 0] > 0).sum())
        t = buf[:n].astype(np.int64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        cols = [0, 1, 2, 3, 4, 5, 6, 7] if fused else [0, 1, 5, 6, 7]
        if fused and os.environ.get("TRACE_SPLIT"):         # split field: 9 chunk sums, 8 chunk scan
            cols = [0, 1, 2, 3, 9, 8, 4, 5, 6, 7]
        if s in (1, 2) and not os.environ.get("TRACE_SPLIT"):
            end = rel[:, 7]
            sm = buf[:n, 8].astype(int)
            nvt = 8
            blk = np.arange(n)
            print("  slowest 12 CTAs (block, sm, vtile, strip, end):",
                  [(int(b), int(sm[b]), int(b % nvt), int(b // nvt), round(float(end[b]), 1)) for b in np.argsort(end)[-12:]])
            print("  end by vtile:", [round(float(np.median(end[blk % nvt == v])), 1) for v in range(nvt)],
                  "max", [round(float(np.max(end[blk % nvt == v])), 1) for v in range(nvt)])
            print("  end by sm<74:", round(float(np.median(end[sm < 74])), 1), round(float(np.median(end[sm >= 74])), 1),
                  "ctas per sm", np.bincount(np.bincount(sm)))
            print("  end pct 50/75/90/95/99/100:", [round(float(np.percentile(end, p)), 1) for p in (50, 75, 90, 95, 99, 100)])
        print(f"fused={fused} stage {s} ctas {n}: " + "  ".join(
            f"{c}:[{np.percentile(rel[:, c], 0):.1f} {np.percentile(rel[:, c], 50):.1f} {np.percentile(rel[:, c], 100):.1f}]"
            for c in cols))

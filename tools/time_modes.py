"""Per-launch CUDA-event times of the C4 step in the fused (field solve inside the stage kernel)
and unfused (circulant kernel + stage kernel) modes: how much the fused prologue costs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1204_3853_b200.solver import UniformVlasov1D  # noqa: E402

w = inputs.get(sys.argv[1] if len(sys.argv) > 1 else "C4")
dt = inputs.fixed_dt(w)
out = {}
for fused in (True, False):
    S = UniformVlasov1D(w.ncells, w.lower, inputs.spacing(w), inputs.level0_boxes(w), inputs.background_profile(w),
                        fused=fused)
    S.set_state(inputs.initial_cell_averages(w))
    for _ in range(3):
        S.step(dt)
    n = 20
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(4 * n)]
    with torch.cuda.stream(S.stream):
        for it in range(n):
            for s in (1, 2, 3, 4):
                e = ev[it * 4 + s - 1]
                e[0].record(S.stream)
                S.field_launch(s)
                e[1].record(S.stream)
                S.stage_launch(s, dt)
                e[2].record(S.stream)
    S.stream.synchronize()
    field = [sum(ev[it * 4 + s][0].elapsed_time(ev[it * 4 + s][1]) for it in range(n)) / n * 1e3 for s in range(4)]
    stage = [sum(ev[it * 4 + s][1].elapsed_time(ev[it * 4 + s][2]) for it in range(n)) / n * 1e3 for s in range(4)]
    out["fused" if fused else "unfused"] = {"field_us": [round(x, 1) for x in field], "stage_us": [round(x, 1) for x in stage]}
print(json.dumps(out))

"""Write tests/golden/c3_100_steps.npz: the oracle's C3 run (BASELINE.json C3: base 128x256,
ratio (4,4) 32x32 tiles, tol 0.005, tag buffer 1, regrid every 10 steps, fixed dt) for 100 RK4
steps, with the fine box lists and the dilated level-0 tags of every regrid.

Calls only oracle/ and inputs/ (through tests/amr_drivers.py, the oracle-side driver of the GPU
parity tests); the oracle takes about an hour for this run, which is why the GPU test reads the
stored result instead of recomputing it.  Usage: python tools/gen_golden_c3.py [nsteps]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import amr_drivers as drv  # noqa: E402
import inputs  # noqa: E402


def main():
    nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    w = inputs.get("C3")
    a = w.amr
    dt = inputs.fixed_dt(w, a["ratio"])
    log = []
    t0 = time.time()
    H, data, E_bc = drv.c3_run(w, nsteps, a["regrid"], dt, a["tol"], a["buffer"], a["ratio"], a["tile"], log=log)
    out = {"nsteps": np.int64(nsteps), "dt": np.float64(dt), "seconds": np.float64(time.time() - t0)}
    for k, (n, nb, tags) in enumerate(log):
        out[f"regrid{k}_step"] = np.int64(n)
        out[f"regrid{k}_boxes"] = np.asarray(nb, dtype=np.int32).reshape(-1, 2, 2)
        out[f"regrid{k}_tags"] = np.packbits(np.asarray(tags, dtype=bool).ravel())
    out["nregrids"] = np.int64(len(log))
    for l, lvl in enumerate(data):
        out[f"level{l}_npatches"] = np.int64(len(lvl))
        for p, arr in enumerate(lvl):
            out[f"level{l}_patch{p}"] = np.ascontiguousarray(arr[2:-2, 2:-2])
    for l, E in enumerate(E_bc):
        out[f"E{l}"] = np.asarray(E)
    path = os.path.join(ROOT, "tests", "golden", f"c3_{nsteps}_steps.npz")
    np.savez_compressed(path, **out)
    print(path, f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()

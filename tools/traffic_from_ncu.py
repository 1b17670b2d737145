"""Write profiles/stage_traffic_<workload>.json (DRAM bytes per RK4 step of the stage kernels, read
by bench.py's roofline.traffic) from an `ncu --set full` capture of the 4 stage launches of one step.
usage: traffic_from_ncu.py REP CELLS WORKLOAD KERNEL_SUBSTRING"""
import csv
import io
import json
import os
import subprocess
import sys

rep = sys.argv[1]
cells = int(sys.argv[2]) if len(sys.argv) > 2 else 2048 * 4096
wname = sys.argv[3] if len(sys.argv) > 3 else "C4"
kname = sys.argv[4] if len(sys.argv) > 4 else "k_stage_1d1v"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
kn = hdr.index("Kernel Name")
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}
tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def val(r, key, table):
    i = hdr.index(key)
    return float(r[i]) * table[units[i]]


per = []
for r in rows[2:]:
    if kname not in r[kn]:
        continue
    i = hdr.index("lts__t_sectors_srcunit_tex_op_write.sum")
    l2w = float(r[i].replace(",", "")) * 32.0          # sectors the SMs wrote into L2 (32 B each)
    per.append({"kernel": r[kn][:60], "dram_read_bytes": val(r, "dram__bytes_read.sum", scale),
                "dram_write_bytes": val(r, "dram__bytes_write.sum", scale),
                "l2_write_bytes_from_sm": l2w,
                "duration_us": val(r, "gpu__time_duration.sum", tscale)})
per = per[:4]
# Traffic charged to a launch: its DRAM reads plus every sector it dirtied in L2.  ncu's
# dram__bytes_write.sum only sees write-backs that happen while the kernel runs; a streaming kernel
# whose output (67-134 MB) largely fits the 126 MB L2 leaves most of it dirty at exit and it is
# written back during later launches.  Each dirtied sector is written to DRAM exactly once (the
# kernels write every output sector once), so reads + L2 writes is the launch's DRAM traffic.
tot = sum(p["dram_read_bytes"] + max(p["dram_write_bytes"], p["l2_write_bytes_from_sm"]) for p in per)
if len(per) != 4:
    sys.exit(f"need the 4 stage launches of one step, found {len(per)}")
res = {"source": f"ncu --set full --clock-control none, {len(per)} stage launches of one {wname} RK4 step ({rep})",
       "bytes_per_step": tot, "bytes_per_step_per_cell": tot / cells, "algorithmic_bytes_per_step_per_cell": 96,
       "definition": "per launch: dram__bytes_read.sum + max(dram__bytes_write.sum, 32 x "
                     "lts__t_sectors_srcunit_tex_op_write.sum) (every sector the kernel dirties in L2 is "
                     "written back once, during or after the launch)",
       "per_launch": per}
dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"stage_traffic_{wname}.json")
json.dump(res, open(dst, "w"), indent=1)
print(json.dumps(res, indent=1))

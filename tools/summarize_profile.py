"""Numbers for profiles/r1_summary.md from a tools/gpu_profile.sh run:
python tools/summarize_profile.py gpurun_out/prof_launches.csv gpurun_out/prof_full.ncu-rep"""
import csv
import subprocess
import sys
from collections import OrderedDict

launches, rep = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = OrderedDict()
for r in rows[1:]:
    d.setdefault(int(r[ii]), {"k": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
ids = sorted(d)
# one full step: from the 2nd-to-last forward GEMM up to the next forward GEMM
fw = [i for i in ids if "k_gemmq<0>" in d[i]["k"]]
# a steady-state step: the forward follows the previous step's fixup (not a call's prologue)
pairs = [(x, y) for x, y in zip(fw, fw[1:])
         if x - 1 in d and "fixup" in d[x - 1]["k"] and not any("k_vmax" in d[i]["k"] for i in ids if x <= i < y)]
a, b = pairs[-1]
tot = sum(d[i]["gpu__time_duration.sum"] for i in ids if a <= i < b)
print(f"one step in the ncu list (IDs {a}..{b - 1}): {tot / 1e6:.3f} ms")
agg = OrderedDict()
for i in ids:
    if a <= i < b:
        name = d[i]["k"].split("(")[0].replace("void ", "").replace("sos::", "")
        e = agg.setdefault(name, [0.0, 0.0, 0])
        e[0] += d[i]["gpu__time_duration.sum"]
        e[1] += d[i].get("dram__bytes_read.sum", 0) + d[i].get("dram__bytes_write.sum", 0)
        e[2] += 1
for name, (t, by, n) in agg.items():
    print(f"  {name:28s} x{n}  {t / 1e6 / n:8.3f} ms/launch  share {t / tot * 100:5.1f} %  DRAM {by / n / 1e9:7.2f} GB/launch")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, u = rr[0], rr[1]
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second", "lts__t_sector_hit_rate.pct",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "smsp__inst_executed_op_global_red.sum",
        "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors.sum"]
for r in rr[2:]:
    print("---", r[h.index("Kernel Name")][:40])
    for w in want:
        if w in h:
            print(f"  {w}: {r[h.index(w)]} {u[h.index(w)]}")

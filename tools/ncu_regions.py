"""Instruction shares of K2+K3 by source region: the ncu SASS source page
(instructions executed per address) joined with nvdisasm -g line info.

Usage: python tools/ncu_regions.py REPORT_SASS.csv CUBIN MANGLED_NAME
(REPORT_SASS.csv = `ncu -i rep --page source --csv --print-source sass`)."""
import csv, re, subprocess, sys
from collections import defaultdict

sass_csv, cubin, fun = sys.argv[1:4]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
lines = dis.splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith("//----") and ".text." + fun + " " in ln)
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("//----")), len(lines))
off2line, cur = {}, None
for ln in lines[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ia, ie, iw = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(rows[2][ia], 16)
per_line = defaultdict(lambda: [0, 0])
tot = [0, 0]
for r in rows[2:]:
    if len(r) <= ie:
        continue
    off = int(r[ia], 16) - base
    n, w = int(r[ie] or 0), int(r[iw] or 0)
    key = off2line.get(off, ("?", 0))
    per_line[key][0] += n
    per_line[key][1] += w
    tot[0] += n
    tot[1] += w


def region(f, l):
    """Code regions of k23.cuh / d4orm_common.cuh (line ranges of the v11 sources)."""
    if f == "d4orm_common.cuh":
        if 140 <= l <= 164: return "noise: Philox4x32-10"
        if 165 <= l <= 193: return "noise: Box-Muller"
        if 100 <= l <= 135: return "packed FP2 ops (pair/obstacle tests, goal)"
        if 60 <= l <= 99: return "rollout: RK4"
        return "other (common)"
    if f == "k23.cuh":
        if 105 <= l <= 200: return "fitness: tile helpers"
        if 203 <= l <= 208: return "fitness: obstacle range lookup"
        if 241 <= l <= 336: return "fitness: diagonal tiles, extents + obstacles"
        if 337 <= l <= 374: return "fitness: diagonal tiles, inner pairs"
        if 377 <= l <= 426: return "fitness: off-diagonal tile pairs"
        if 485 <= l <= 631: return "rollout: controls, clamp, goal, z/position stores"
        if 783 <= l <= 800: return "chunk ranking"
        if 881 <= l <= 942: return "phase-B glue + final reduction"
        return "other (setup, barriers)"
    return "intrinsics (" + f + ")"


print(f"total warp instructions {tot[0]:.4g}, stall samples {tot[1]}")
if "--regions" in sys.argv:
    agg = defaultdict(lambda: [0, 0])
    for (f, l), (n, w) in per_line.items():
        a = agg[region(f, l)]
        a[0] += n
        a[1] += w
    for r, (n, w) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"| {r} | {100*n/tot[0]:.1f} % | {100*w/tot[1]:.1f} % |")
else:
    for (f, l), (n, w) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:60]:
        print(f"{f:22s}{l:5d}  inst {100*n/tot[0]:5.2f}%  samples {100*w/tot[1]:5.2f}%")

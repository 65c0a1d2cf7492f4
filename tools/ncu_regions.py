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


ROOT = __import__("pathlib").Path(__file__).resolve().parent.parent / "paper_2503_12204_b200" / "csrc"
# region = the last anchor (a source substring) at or above the line
ANCHORS = {
    "d4orm_common.cuh": [("enum Kind", "other (common)"), ("fast_sincos", "rollout: RK4"),
                         ("detail::rk4_with", "rollout: RK4"), ("packed f32x2", "packed FP2 ops (tests, goal, controls)"),
                         ("Philox noise", "noise: Philox4x32-10"), ("(2k+1)", "noise: Box-Muller")],
    "k23.cuh": [("namespace d4k", "other (setup, barriers)"), ("fp32 tiles", "fitness (tiles): helpers"),
                ("Obstacle index range", "fitness (tiles): obstacle range lookup"),
                ("One (sample, t) item in fp32", "fitness (tiles): diagonal tiles + obstacles"),
                ("pairs inside tile a", "fitness (tiles): diagonal inner pairs"),
                ("const int n_off", "fitness (tiles): off-diagonal tile pairs"),
                ("---- fp32 pair-list path", "fitness (pair list): block tests"),
                ("One (sample, t) item of the pair-list", "fitness (pair list): boxes + self pairs"),
                ("pair-pair blocks (l, l + d", "fitness (pair list): pair-pair liveness + loop"),
                ("obstacles: pair boxes vs", "fitness (pair list): obstacles"),
                ("One (sample, t) item in fp64", "fitness fp64"),
                ("fp32 fused rollout (phase A)", "rollout: controls, clamp, goal, stores, boxes"),
                ("Chunk sort key", "chunk ranking"), ("One robot's `nsteps` steps", "rollout: controls, clamp, goal, stores, boxes"),
                ("Exact replay of a chunk", "rollout: replay"), ("__launch_bounds__", "other (setup, barriers)"),
                ("rank the sample's robots", "chunk ranking"), ("phase A: integrate", "rollout: controls, clamp, goal, stores, boxes"),
                ("phase B: fitness", "phase-B glue + final reduction")],
    "k_pl32.cuh": [("namespace d4k", "other (setup, barriers)"),
                   ("Half h of one (sample, 32-step window) item", "fitness (pair list): boxes + self pairs"),
                   ("pair-pair blocks (l, l + d mod 32) for this half", "fitness (pair list): pair-pair liveness + loop"),
                   ("obstacles o ≡ h (mod 2): pair boxes", "fitness (pair list): obstacles"),
                   ("template <int KIND, bool RFULL>", "other (setup, barriers)"),
                   ("every 64 steps: rank the sample", "chunk ranking"),
                   ("phase A: integrate the window", "rollout: controls, clamp, goal, stores, boxes"),
                   ("phase B: this warp's half", "phase-B glue + final reduction")],
}
_tables = {}


def region(f, l):
    if f not in ANCHORS:
        return "intrinsics (" + f + ")"
    if f not in _tables:
        lines = (ROOT / f).read_text().splitlines()
        marks = []
        for sub, name in ANCHORS[f]:
            for i, ln in enumerate(lines, 1):
                if sub in ln:
                    marks.append((i, name))
                    break
        _tables[f] = sorted(marks)
    name = "other"
    for i, nm in _tables[f]:
        if i <= l:
            name = nm
    return name


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

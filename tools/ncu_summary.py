"""Summarise an `ncu --set full` report of one denoising step (tools/ncu_k23.py)
into a markdown table and profiles/ncu_summary.json (the bench line's
roofline.ncu / traffic for that workload).

Usage: python tools/ncu_summary.py REPORT.ncu-rep WORKLOAD_NAME OUT.md [raw.csv]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

METRICS = {
    "dur_us": "gpu__time_duration.sum",
    "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "fma_inst_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "alu_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "warps_per_sm": "sm__warps_active.avg.per_cycle_active",
    "regs": "launch__registers_per_thread",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "inst": "smsp__inst_executed.sum",
    "ffma_thread_inst": "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
}


def load(rep):
    if str(rep).endswith(".csv"):  # already exported on the GPU box (`ncu -i rep --page raw --csv`)
        out = Path(rep).read_text()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "?")}
        for key, m in METRICS.items():
            v = d.get(m)
            if v in (None, "", "n/a"):
                k[key] = None
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                k[key] = None
                continue
            unit = u.get(m, "")
            if key == "dur_us":
                x = x * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                         "s": 1e6, "second": 1e6}.get(unit, 1.0)
            if key.startswith("dram"):
                x = x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
                         "GB": 1e9}.get(unit, 1)
            k[key] = x
        res.append(k)
    return out, res


def main():
    rep, name, md = sys.argv[1:4]
    raw, ks = load(rep)
    if len(sys.argv) > 4:
        Path(sys.argv[4]).write_text(raw)
    lines = [f"# ncu --set full, one {name} denoising step (`{Path(rep).name}`)", "",
             "| kernel | µs | issue % | FMA pipe cycles % | FMA pipe inst % | ALU % | XU % | LSU % | warps/SM | regs | DRAM read + write |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for k in ks:
        nm = k["kernel"].split("(")[0][:60]
        f = lambda v, p=1: "–" if v is None else f"{v:.{p}f}"
        dram = (k["dram_read"] or 0) + (k["dram_write"] or 0)
        lines.append(f"| `{nm}` | {f(k['dur_us'])} | {f(k['issue_pct'])} | {f(k['fma_pct'])} | {f(k['fma_inst_pct'])} | "
                     f"{f(k['alu_pct'])} | {f(k['xu_pct'])} | {f(k['lsu_pct'])} | {f(k['warps_per_sm'])} | "
                     f"{f(k['regs'], 0)} | {dram / 1e6:.1f} MB |")
    Path(md).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))
    k23 = next((k for k in ks if "rollout_fitness" in k["kernel"]), None)
    if k23:
        sj = ROOT / "profiles" / "ncu_summary.json"
        data = json.loads(sj.read_text()) if sj.exists() else {}
        kname = k23["kernel"].split("(")[0].replace("void ", "").strip()
        data[name] = {"kernel": f"{kname} (K2+K3)", "issue_active_pct": k23["issue_pct"],
                      "fma_pipe_cycles_pct": k23["fma_pct"], "fma_pipe_inst_pct": k23["fma_inst_pct"],
                      "alu_pipe_pct": k23["alu_pct"],
                      "xu_pipe_pct": k23["xu_pct"], "warps_per_sm": k23["warps_per_sm"], "registers": k23["regs"],
                      "duration_us_cold": k23["dur_us"], "source": f"profiles/{Path(md).name}"}
        sj.write_text(json.dumps(data, indent=1) + "\n")
        tj = ROOT / "profiles" / "traffic.json"
        t = json.loads(tj.read_text()) if tj.exists() else {}
        t[name] = (k23["dram_read"] or 0) + (k23["dram_write"] or 0)
        t.pop("_source", None)
        t.setdefault("_sources", {})[name] = (f"profiles/{Path(md).name} (ncu --set full, one launch of "
                                              f"{kname}: dram__bytes_read.sum + dram__bytes_write.sum)")
        tj.write_text(json.dumps(t, indent=1) + "\n")


if __name__ == "__main__":
    main()

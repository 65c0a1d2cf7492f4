"""Generate tests/golden/golden.{npz,json} from the REFERENCE's own code
(oracle/_ref/libd4orm_ref.so = /root/reference/proj/src compiled unchanged).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures pin the oracle on machines without /root/reference."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Reference, make_config  # noqa: E402
from paper_2503_12204_b200 import scenarios as S  # noqa: E402

ref = Reference()
out, meta = {}, {"normal_seeds": [0, 1, 77, 2**40 + 3], "normal_count": 513, "cases": [],
                 "source": "oracle/_ref (reference proj/src compiled unchanged)"}
for s in meta["normal_seeds"]:
    out[f"normal_{s}"] = ref.normal_fill(s, meta["normal_count"])
rng = np.random.default_rng(2024)
for cfg_idx, horizon, steps, batch in [(1, 64, 3, 32), (2, 24, 2, 16), (3, 24, 2, 16), (4, 24, 2, 16), (5, 6, 2, 8)]:
    p = S.baseline_config(cfg_idx).problem.with_horizon(horizon)
    cid = f"C{cfg_idx}"
    u = rng.normal(size=(p.horizon, p.robots, p.du)) * 1.5
    st, ct = ref.rollout(p, u)
    base = ct[:-1].copy()
    v, tr = ref.run_denoising(p, base, make_config(steps, batch, seed=cfg_idx))
    out.update({f"{cid}_u": u, f"{cid}_states": st, f"{cid}_reward": np.array(ref.total_reward(p, st)),
                f"{cid}_base": base, f"{cid}_variable": v, f"{cid}_trace": np.array(tr)})
    meta["cases"].append({"id": cid, "config": cfg_idx, "horizon": horizon, "steps": steps, "batch": batch,
                          "seed": cfg_idx})
np.savez_compressed(Path(__file__).parent / "golden.npz", **out)
(Path(__file__).parent / "golden.json").write_text(json.dumps(meta, indent=1))
print("wrote", len(out), "arrays")

"""CPU model of the throughput-mode noise (test infrastructure only).

The fp32 path draws its normals on the device (d4orm_common.cuh: Philox,
u01_open, box_muller, philox_normals; d4orm_kernels.cuh K1 layout).  This
module restates that generator in numpy so the GPU bits can be checked:

* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy
  as 1, 2, 3", SC'11): multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key bumps
  0x9E3779B9 / 0xBB67AE85.  Pinned by the published known-answer vectors
  below (Random123 kat_vectors, philox4x32 with 10 rounds).
* Counter mapping: normals of (seed_it, step i, sample m, robot k) form one
  sequence n = t·du + d; group g = n // 4 is Philox(counter = (k, g, m_hi,
  m_lo), key = mix_seed(seed_it, i) split lo/hi), lane n % 4.
* Uniforms from the top 23 bits: u = (2j+1)·2^-24 for j = x >> 9 (exact);
  angle 2π·j·2^-23.  Box-Muller (r cos θ, r sin θ) on the lane pairs (0,1) and
  (2,3); the device evaluates log2 / sqrt / sincos on the MUFU unit
  (approximate), so normals agree to ~1e-5 while the integer stream is exact.
"""
from __future__ import annotations

import numpy as np

from paper_2503_12204_b200.scenarios import mix_seed

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)

# (counter, key) -> output, Philox4x32-10 (Random123 known-answer vectors)
KAT = [
    ((0x00000000, 0x00000000, 0x00000000, 0x00000000), (0x00000000, 0x00000000),
     (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF), (0xFFFFFFFF, 0xFFFFFFFF),
     (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


def philox4x32(c0, c1, c2, c3, k0, k1, rounds: int = 10):
    """Vectorised Philox4x32 over numpy uint32-valued arrays (broadcasting)."""
    c = [np.asarray(v, dtype=np.uint64) & MASK32 for v in (c0, c1, c2, c3)]
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for _ in range(rounds):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = [((p1 >> np.uint64(32)) ^ c[1] ^ np.uint64(k0)) & MASK32, p1 & MASK32,
             ((p0 >> np.uint64(32)) ^ c[3] ^ np.uint64(k1)) & MASK32, p0 & MASK32]
        k0 = (k0 + W0) & 0xFFFFFFFF
        k1 = (k1 + W1) & 0xFFFFFFFF
    return [v.astype(np.uint32) for v in c]


def step_key(seed_it: int, step: int) -> tuple[int, int]:
    v = mix_seed(seed_it, step)
    return v & 0xFFFFFFFF, v >> 32


def philox_words(seed_it: int, step: int, m0: int, count: int, R: int, T: int, du: int) -> np.ndarray:
    """Raw Philox words, [count][R][G][4] with G = ceil(T·du/4)."""
    G = (T * du + 3) // 4
    k0, k1 = step_key(seed_it, step)
    m = (np.arange(count, dtype=np.uint64) + np.uint64(m0))[:, None, None]
    k = np.arange(R, dtype=np.uint64)[None, :, None]
    g = np.arange(G, dtype=np.uint64)[None, None, :]
    out = philox4x32(k + 0 * m + 0 * g, g + 0 * m + 0 * k, (m >> np.uint64(32)) + 0 * k + 0 * g,
                     (m & MASK32) + 0 * k + 0 * g, k0, k1)
    return np.stack(out, axis=-1)


def normals(seed_it: int, step: int, m0: int, count: int, R: int, T: int, du: int) -> np.ndarray:
    """Normals in the K1 layout [count][T][R][du] (float64 evaluation)."""
    w = philox_words(seed_it, step, m0, count, R, T, du).astype(np.uint64)
    j = (w >> np.uint64(9)).astype(np.float64)
    u = (2.0 * j + 1.0) * 2.0 ** -24            # radius uniform, (0, 1)
    th = 2.0 * np.pi * j * 2.0 ** -23           # angle
    r01 = np.sqrt(-2.0 * np.log(u[..., 0]))
    r23 = np.sqrt(-2.0 * np.log(u[..., 2]))
    z = np.stack([r01 * np.cos(th[..., 1]), r01 * np.sin(th[..., 1]),
                  r23 * np.cos(th[..., 3]), r23 * np.sin(th[..., 3])], axis=-1)  # [count][R][G][4]
    count_, R_, G, _ = z.shape
    seq = z.reshape(count_, R_, G * 4)[:, :, : T * du].reshape(count_, R_, T, du)
    return np.ascontiguousarray(seq.transpose(0, 2, 1, 3))

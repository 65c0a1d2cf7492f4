"""CPU, world_size 2 over gloo: the sample-sharded step protocol (reward
all-gather → identical weights on every rank → chunk-tree partials → root
all-gather → same tree) gives a bitwise identical denoised variable on every
rank and for world 1 and 2, and matches the reference's sequential step.  The
per-rank compute here is the CPU oracle (test infrastructure); on the GPUs the
same protocol runs inside the C-ABI with NCCL (csrc/d4orm_cuda.cu)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_12204_b200 import scenarios as S
from paper_2503_12204_b200.sharding import CHUNK, chunk_partials, pairwise_tree, shard_range

N, I, SEED = 8, 5, 3
M = 1024


def problem():
    return S.baseline_config(1).problem.with_horizon(12)


def local_step(oracle, p, base, var, rank, world, gather, M=M):
    """One denoising step i=I from `var`, samples [m0, m0+Ml) computed here."""
    ab, _ = oracle.make_schedule(N, 0.05)
    ms, sd = 1 / math.sqrt(ab[I]), math.sqrt(1 / ab[I] - 1)
    m0, Ml = shard_range(M, world, rank)
    z = oracle.step_noise(SEED, I, m0, Ml, p.elems)
    samples = ms * var.reshape(1, -1) + sd * z
    rewards = np.empty(Ml)
    for j in range(Ml):
        st, _ = oracle.rollout(p, base.reshape(-1) + samples[j])
        rewards[j] = oracle.total_reward(p, st)[0]
    all_rewards = gather(rewards)                      # ncclAllGather(rewards)
    w = oracle.score_weights(all_rewards, 0.1)         # identical on every rank
    root = pairwise_tree(chunk_partials(samples, w[m0:m0 + Ml]))
    roots = gather(root.reshape(1, -1)).reshape(world, -1)  # ncclAllGather(roots)
    return math.sqrt(ab[I - 1]) * pairwise_tree(list(roots)), all_rewards


def _worker(rank, world, port, q, M=M):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    oracle = Oracle()
    p = problem()
    rng = np.random.default_rng(0)
    base = 0.2 * rng.normal(size=p.elems)
    var = 0.1 * rng.normal(size=p.elems)

    def gather(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t)
        return torch.cat(out).numpy()

    v, r = local_step(oracle, p, base, var, rank, world, gather, M)
    q.put((rank, v, r))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world,M", [(2, 1024), (3, 1536)])
def test_sharded_step_is_world_invariant(oracle, world, M):
    """world 3 at M = 1536: two chunks per rank (a power of two), so the three
    roots are subtrees of the single-GPU tree although G is not."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, M)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort(key=lambda t: t[0])
    v0 = res[0][1]
    for r in range(1, world):
        np.testing.assert_array_equal(v0, res[r][1])    # every rank holds the same variable

    # world = 1 with the same protocol: bitwise the same result
    p = problem()
    rng = np.random.default_rng(0)
    base = 0.2 * rng.normal(size=p.elems)
    var = 0.1 * rng.normal(size=p.elems)
    v_single, r_single = local_step(oracle, p, base, var, 0, 1, lambda a: np.asarray(a, dtype=np.float64), M)
    np.testing.assert_array_equal(v0, v_single)
    np.testing.assert_array_equal(res[0][2], r_single)

    # and the reference's own sequential step (mc_average in ascending m) to rounding
    ab, _ = oracle.make_schedule(N, 0.05)
    from oracle.oracle import make_config
    v_ref, r_ref, _, _ = oracle.denoise_step(p, base, var, ab, make_config(N, M, seed=SEED), I)
    np.testing.assert_array_equal(r_single, r_ref)
    np.testing.assert_allclose(v_single, v_ref.reshape(-1), rtol=1e-12, atol=1e-14)


def test_shard_ranges():
    assert shard_range(262144, 8, 3) == (3 * 32768, 32768)
    with pytest.raises(ValueError):
        shard_range(1000, 3, 0)
    with pytest.raises(ValueError):
        shard_range(1024, 8, 0)  # 128 per rank is not a whole chunk
    with pytest.raises(ValueError, match="power of two"):
        shard_range(1536, 2, 0)  # 3 chunks per rank: not one subtree of the single-GPU tree
    assert shard_range(1536, 3, 2) == (1024, 512)
    # why: the single tree over 6 chunks groups (c0..c3)(c4,c5); ranks of 3 chunks would group (c0..c2)(c3..c5)
    parts6 = [float(x) for x in np.random.default_rng(2).normal(size=6)]
    assert pairwise_tree(parts6) == ((parts6[0] + parts6[1]) + (parts6[2] + parts6[3])) + (parts6[4] + parts6[5])
    parts = [float(x) for x in np.random.default_rng(1).normal(size=16)]
    full = pairwise_tree(parts)
    for g in (2, 4, 8):
        roots = [pairwise_tree(parts[r * 16 // g:(r + 1) * 16 // g]) for r in range(g)]
        assert pairwise_tree(roots) == full
    parts24 = [float(x) for x in np.random.default_rng(3).normal(size=24)]
    for g in (3, 6, 12):  # 8, 4, 2 leaves per rank
        roots = [pairwise_tree(parts24[r * 24 // g:(r + 1) * 24 // g]) for r in range(g)]
        assert pairwise_tree(roots) == pairwise_tree(parts24)
    assert CHUNK == 256

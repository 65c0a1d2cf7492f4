"""The C-ABI's world > 1 path on the B200: ranks as separate processes.

Each rank is its own process with its own context (d4orm_cuda_create(device,
rank, world, ...)), owning the contiguous samples [r·M/G, (r+1)·M/G); the
step's two all-gathers (rewards → K4 on the full vector, chunk-tree roots →
the top of the pairwise tree) run either over NCCL (one GPU per rank: skipped
when fewer GPUs are visible) or through the host exchange function
(d4orm_cuda_set_exchange_fn) over torch.distributed gloo.  The host exchange
lets G ranks share one GPU without any kernel waiting on another rank (each
exchange is a blocking host call between kernels), so the sharded code path
— shard offsets, global Philox indices, the reward gather, the per-rank tree
roots, the replicated K4/K5b — runs on the real kernels here.

Expected: every rank returns the same variable / trace / solve
result, bitwise equal to the single-GPU run, for G = 2 and 3 (a rank must own
256 × a power-of-two samples; G itself may be anything).
"""
import os
import socket

import numpy as np
import pytest

import paper_2503_12204_b200 as d4
from paper_2503_12204_b200 import scenarios as S

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(name):
    if name == "C5":
        return S.baseline_config(5).problem.with_horizon(64)
    return S.baseline_config(2).problem.with_horizon(48)


def _workload(g, p, M, oracle_noise=None):
    """Everything the sharded path runs: a Philox denoising step, a short
    run_denoising, a 2-iteration solve, MPPI and CEM, and a host-noise fp64
    run (each rank receives its own slice of the provider's noise)."""
    out = {}
    rng = np.random.default_rng(3)
    base = np.zeros((p.horizon, p.robots, p.du))
    var = 0.2 * rng.normal(size=base.shape)
    cfg = d4.DenoiserConfig(steps=10, batch=M, seed=5)
    g.set_options(d4.PREC_F32, d4.NOISE_PHILOX, True)
    g.set_problem(p)
    out["step"] = g.denoise_step(base, var, 10, cfg)
    out["run"] = g.run_denoising(base, d4.DenoiserConfig(steps=4, batch=M, seed=6))
    sr = g.solve(d4.DenoiserConfig(steps=3, batch=M, seed=7), max_iterations=2, stop_on_success=False)
    out["solve"] = ([x[:3] for x in sr.per_iteration], sr.best_states, sr.traces)
    mr = g.mppi_solve(batch=M, iterations=2, seed=3, stop_on_success=False)
    out["mppi"] = ([x[:3] for x in mr.per_iteration], mr.best_controls)
    cr = g.cem_solve(batch=M, iterations=2, seed=3, stop_on_success=False)
    out["cem"] = ([x[:3] for x in cr.per_iteration], cr.best_controls)
    g.set_options(d4.PREC_F64, d4.NOISE_HOST, True)
    g.set_noise_provider(lambda step, m0, count, elems: np.sin(
        0.001 * (np.arange(m0, m0 + count)[:, None] * elems + np.arange(elems)[None, :]) + step))
    out["host64"] = g.run_denoising(base, d4.DenoiserConfig(steps=3, batch=M, seed=1))
    return out


def _worker(rank, world, port, q, name, M):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def exchange(local: bytes) -> bytes:
        t = torch.frombuffer(bytearray(local), dtype=torch.uint8)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return b"".join(x.numpy().tobytes() for x in parts)

    try:
        p = _problem(name)
        g = d4.GpuDenoiser(device=0, rank=rank, world=world, exchange=exchange)
        res = _workload(g, p, M)
        assert g.launches_per_step() >= 5
        g.close()
        q.put((rank, res, None))
    except Exception as e:  # reported to the parent
        q.put((rank, None, repr(e)))
    dist.barrier()
    dist.destroy_process_group()


def _run_ranks(world, name, M):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, name, M)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
    res.sort(key=lambda t: t[0])
    for r, _, err in res:
        assert err is None, f"rank {r}: {err}"
    return [x[1] for x in res]


def _assert_same(a, b, path=""):
    if isinstance(a, dict):
        assert a.keys() == b.keys()
        for k in a:
            _assert_same(a[k], b[k], f"{path}.{k}")
    elif isinstance(a, (list, tuple)):
        assert len(a) == len(b), path
        for i, (x, y) in enumerate(zip(a, b)):
            _assert_same(x, y, f"{path}[{i}]")
    elif isinstance(a, np.ndarray):
        np.testing.assert_array_equal(a, b, err_msg=path)
    else:
        assert a == b, (path, a, b)


@pytest.mark.parametrize("world,name,M", [(2, "C2", 8192), (3, "C2", 3 * 2048), (2, "C5", 8192)])
def test_sharded_ranks_equal_single_gpu(world, name, M):
    single = _workload(d4.GpuDenoiser(device=0), _problem(name), M)
    ranks = _run_ranks(world, name, M)
    for r, res in enumerate(ranks):
        _assert_same(res, single, f"rank{r}")


def test_sharded_batch_rule():
    """A rank must own 256 × 2^k samples (else its partials are not one subtree
    of the single-GPU tree and the result would depend on G)."""
    def exchange(local):
        return local * 2
    g = d4.GpuDenoiser(S.baseline_config(1).problem, device=0, rank=0, world=2, exchange=exchange)
    base = np.zeros((64, 4, 2))
    with pytest.raises(ValueError, match="must be 256 x a power of two"):
        g.run_denoising(base, d4.DenoiserConfig(steps=2, batch=1536))
    with pytest.raises(ValueError, match="not divisible by world"):
        g.run_denoising(base, d4.DenoiserConfig(steps=2, batch=1025))
    g.close()
    h = d4.GpuDenoiser(S.baseline_config(1).problem, device=0, rank=1, world=2)
    with pytest.raises(ValueError, match="needs an NCCL id or an exchange fn"):
        h.run_denoising(base, d4.DenoiserConfig(steps=2, batch=1024))
    h.close()


def _nccl_worker(rank, world, port, q):
    import ctypes as C
    import torch.distributed as dist
    from paper_2503_12204_b200._lib import lib
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    obj = [None]
    if rank == 0:
        buf = C.create_string_buffer(128)
        assert lib().d4orm_cuda_nccl_id(buf) == 0
        obj = [bytes(buf.raw)]
    dist.broadcast_object_list(obj, src=0)
    try:
        g = d4.GpuDenoiser(device=rank, rank=rank, world=world, nccl_id=obj[0])
        q.put((rank, _workload(g, _problem("C5"), 8192), None))
        g.close()
    except Exception as e:
        q.put((rank, None, repr(e)))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_two_gpus_equal_single_gpu():
    """The NCCL transport with one GPU per rank (the bench's multi-GPU path)."""
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip(f"{n} GPU visible: the NCCL transport needs one GPU per rank")
    import torch.multiprocessing as mp
    single = _workload(d4.GpuDenoiser(device=0), _problem("C5"), 8192)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda t: t[0])
    for pr in procs:
        pr.join(timeout=120)
    for r, out, err in res:
        assert err is None, err
        _assert_same(out, single, f"rank{r}")

"""A7: the cross-rank combine of per-shard [logL, g]
vectors, with the CUDA path on both sides, checked against the oracle over
ALL patterns (pytest -m gpu).

Patterns are conditionally independent, so logL and every
gradient entry are sums over pattern shards (Eq. 6 is a column sum,
P:285-291); the combine is one allreduce(sum) of 2N-1 doubles.

  * two processes share cuda:0, each evaluates its shard through the C ABI,
    `allreduce_evaluation` over gloo sums them;
  * a world-size-1 NCCL group with [branch lengths, evaluation, allreduce]
    captured as ONE CUDA graph (the library enqueues into the caller's
    capture), replayed for several branch-length vectors;
  * host staging: set / compute_device / set / compute_device with no host
    synchronisation, queued behind a long kernel, each evaluation sees its
    own branch lengths.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import phylo_synth as ps

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _c17(res, ref):
    el = abs(res[0] - ref["logL"]) / abs(ref["logL"])
    scale = np.maximum(np.abs(ref["grad"]), ref["grad_abs"])
    eg = float(np.max(np.abs(res[1:] - ref["grad"]) / np.where(scale > 0, scale, 1.0)))
    return el, eg


def _problem(kind):
    if kind == "dengue":
        return ps.config1_dengue(N=120, C=301)
    if kind == "codon":
        return ps.config3_yeast(N=16, C=75)
    return ps.config2_mmm(N=24, C=99)


def _gloo_worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2303_04390_b200 as pg
    pb = _problem(kind)
    ev = pg.ShardEvaluation(pb, rank=rank, world=world, device=0)
    out = ev.evaluate()
    ev.stream.synchronize()
    zp = ev.zero_pattern()
    res = out.cpu().numpy().copy()
    if rank == 0:
        q.put((res, zp, ev.hi - ev.lo))
    ev.close()
    dist.barrier()
    dist.destroy_process_group()
    del torch


@pytest.mark.parametrize("kind", ["dengue", "codon", "mmm"])
def test_two_process_shards_allreduce_match_oracle(kind):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res, zp, n0 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    pb = _problem(kind)
    assert 0 < n0 < pb.patterns                     # rank 0 really held a strict shard
    assert zp == -1
    ref = oracle.loglik_grad(pb, threads=8)
    el, eg = _c17(res, ref)
    assert el <= 1e-10 and eg <= 1e-10, (kind, el, eg)


def _nccl_init():
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_free_port())
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    return dist


@pytest.mark.parametrize("kind", ["dengue", "codon"])
def test_nccl_allreduce_captured_in_graph_matches_oracle(kind):
    import torch
    import paper_2303_04390_b200 as pg
    dist = _nccl_init()
    pb = _problem(kind)
    ev = pg.ShardEvaluation(pb, rank=0, world=1, device=0, capture=True)
    assert ev.graph is not None
    rng = np.random.default_rng(11)
    base = pb.branch_lengths.copy()
    for _ in range(3):
        pb.branch_lengths = base * rng.uniform(0.8, 1.2, base.shape)
        out = ev.evaluate(pb.branch_lengths)      # replays [set_bl_device, compute_device, allreduce]
        ev.stream.synchronize()
        res = out.cpu().numpy()
        ref = oracle.loglik_grad(pb, threads=8)
        el, eg = _c17(res, ref)
        assert el <= 1e-10 and eg <= 1e-10, (kind, el, eg)
    ev.close()
    del dist, torch


def test_capture_requires_prior_uploads():
    """Under the caller's capture the library cannot upload: a fresh instance
    reports PG_ERR_SEQUENCE instead of breaking the capture."""
    import torch
    import paper_2303_04390_b200 as pg
    pb = ps.small_problem(8, "hky", R=2, C=20, seed=1, simulate=True)
    inst = pg.from_problem(pb)
    out = torch.zeros(2 * pb.n_tips - 1, dtype=torch.float64, device="cuda")
    g = torch.cuda.CUDAGraph()
    with pytest.raises(pg.PhyloGradError) as ei:
        with torch.cuda.graph(g, stream=inst.stream):
            inst.compute_device(out)
    assert ei.value.code == pg.PG_ERR_SEQUENCE
    inst.close()


def test_host_staging_not_overwritten_by_next_set():
    """set(b1), compute_device(o1), set(b2), compute_device(o2) with no host
    sync, queued behind a ~50 ms kernel: o1 must be the evaluation at b1."""
    import torch
    import paper_2303_04390_b200 as pg
    pb = ps.config1_dengue(N=50, C=120)
    inst = pg.from_problem(pb)
    n = 2 * pb.n_tips - 1
    o1 = torch.zeros(n, dtype=torch.float64, device="cuda")
    o2 = torch.zeros(n, dtype=torch.float64, device="cuda")
    b1 = pb.branch_lengths.copy()
    b2 = b1 * 1.5
    inst.compute()                                   # plan + uploads done
    with torch.cuda.stream(inst.stream):
        torch.cuda._sleep(100_000_000)               # the stream is busy for a while
        inst.set_branch_lengths(b1)
        inst.compute_device(o1)
        inst.set_branch_lengths(b2)
        inst.compute_device(o2)
    inst.stream.synchronize()
    for b, o in ((b1, o1), (b2, o2)):
        pb.branch_lengths = b
        el, eg = _c17(o.cpu().numpy(), oracle.loglik_grad(pb, threads=8))
        assert el <= 1e-10 and eg <= 1e-10
    inst.close()

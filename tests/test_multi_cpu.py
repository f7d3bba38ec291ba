"""N > 1 host logic on CPU: pattern sharding + the allreduce combine (A7),
world size 2 over gloo.  Each rank evaluates its contiguous
pattern shard with the oracle (the CUDA path needs a GPU) and the [logL, g]
vectors are summed with `allreduce_evaluation`, exactly as bench.py does with
NCCL on the GPU path; the result must equal the unsharded evaluation."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2303_04390_b200 as pg
    import phylo_synth as ps
    pb = ps.small_problem(20, "hky", R=4, C=101, seed=3, missing=0.05, simulate=True)
    lo, hi = pg.shard_range(pb.patterns, world, rank)
    r = oracle.loglik_grad(pb, lo, hi)
    out = torch.tensor(np.concatenate([[r["logL"]], r["grad"]]), dtype=torch.float64)
    pg.allreduce_evaluation(out)
    if rank == 0:
        q.put(out.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_allreduce_equals_unsharded():
    import oracle
    import phylo_synth as ps
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    pb = ps.small_problem(20, "hky", R=4, C=101, seed=3, missing=0.05, simulate=True)
    full = oracle.loglik_grad(pb)
    assert abs(res[0] - full["logL"]) <= 1e-12 * abs(full["logL"])
    assert np.max(np.abs(res[1:] - full["grad"]) / full["grad_abs"]) <= 1e-12

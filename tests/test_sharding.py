"""Multi-GPU sharding protocol on CPU with gloo, world size 2.

The engine's sharded mode (pf_create_sharded) gives rank r the subdomains
s % nranks == r and sums every lambda-space partial result over ranks (NCCL on
the device).  Here the same shard plan (the product's pf_shard_plan) and the
same reduction protocol run on CPU: each rank evaluates its subdomains' terms
of the interface operator and of the (unscaled) Dirichlet preconditioner
with the oracle, the partial vectors are all-reduced with gloo, and the sum
must equal the unsharded operator.  The device path is exercised by
tests/test_gpu_parity.py::test_sharded_step_matches_single_engine.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kw, results):
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle_lib as ol
    import paper_2509_06673_b200 as pf
    o = ol.Oracle(**kw)
    plan = pf.shard_plan(o.n_sub, rank, world)
    x = np.random.default_rng(11).uniform(-1, 1, o.n_lambda)
    out = {}
    for which in (0, 1):
        y = torch.from_numpy(o.apply_subset(x, plan, which))
        dist.all_reduce(y)
        out[which] = y.numpy().copy()
    covered = torch.zeros(o.n_sub, dtype=torch.int64)
    covered[plan] += 1
    dist.all_reduce(covered)
    if rank == 0:
        results.put((out[0], out[1], covered.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kw", [
    dict(mesh_n=32, SX=4, SY=4, order=2, steps=1, precond="dirichlet"),            # floating, P|P
    dict(mesh_n=32, SX=1, SY=2, order=1, steps=1, precond="dirichlet"),            # reference layout
])
def test_gloo_two_rank_partial_sums(kw):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import oracle_lib as ol
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kw, q)) for r in range(2)]
    for p in procs:
        p.start()
    yF, yM, covered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert (covered == 1).all()  # every subdomain owned by exactly one rank
    o = ol.Oracle(**kw)
    x = np.random.default_rng(11).uniform(-1, 1, o.n_lambda)
    assert np.linalg.norm(yF - o.apply(x)) <= 1e-13 * np.linalg.norm(yF)
    assert np.linalg.norm(yM - o.precond(x)) <= 1e-13 * np.linalg.norm(yM)


def test_shard_plan_balanced():
    import paper_2509_06673_b200 as pf
    for n_sub, world in ((1024, 8), (64, 4), (2, 2)):
        plans = [pf.shard_plan(n_sub, r, world) for r in range(world)]
        assert sorted(sum(plans, [])) == list(range(n_sub))
        assert max(map(len, plans)) - min(map(len, plans)) <= 1

"""The engine's own sharded path across PROCESSES: two ranks (one process
each, torch.distributed gloo on 127.0.0.1) each own half of the subdomains
(pf_create_sharded) and sum their lambda-space partial results through a host
reducer (pf_set_reducer -> dist.all_reduce).  Only one GPU exists here, so
both processes use it; their kernels never wait on each other -- the exchange
is on the host -- so this checks the protocol, not NCCL or scaling.  Rank 0
compares the step with the unsharded engine."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, port, kw, q):
    import torch
    import torch.distributed as dist

    import paper_2509_06673_b200 as pf
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        op = pf.FetiOperator(rank=rank, nranks=2, **kw)

        def red(buf):
            t = torch.from_numpy(buf)  # shares memory with the engine's host copy
            dist.all_reduce(t)

        op.set_reducer(red)
        x = np.random.default_rng(3).uniform(-1, 1, op.n_lambda)
        y = op.apply(x)
        rep = op.step()
        xs, lam = op.state()
        q.put((rank, op.owned, y, rep["iterations"], [v.copy() for v in xs], lam))
        op.close()
    finally:
        dist.destroy_process_group()


def test_two_process_sharded_step_matches_single_engine():
    import torch.multiprocessing as mp

    import paper_2509_06673_b200 as pf
    kw = dict(pf.BASELINE_CONFIGS["c4"], mesh_n=128, SX=4, SY=4, steps=1)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, port, kw, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r) for r in (q.get(timeout=600) for _ in range(2)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    full = pf.FetiOperator(**kw)
    x = np.random.default_rng(3).uniform(-1, 1, full.n_lambda)
    yf = full.apply(x)
    rf = full.step()
    xf, lf = full.state()
    assert sorted(res[0][1] + res[1][1]) == list(range(16))
    for r in (0, 1):
        _, owned, y, its, xs, lam = res[r]
        assert np.linalg.norm(y - yf) <= 1e-12 * np.linalg.norm(yf)
        assert abs(its - rf["iterations"]) <= 2
        assert np.linalg.norm(lam - lf) <= 1e-9 * np.linalg.norm(lf)
        for s, v in zip(owned, xs):
            assert np.linalg.norm(v - xf[s]) <= 1e-9 * np.linalg.norm(xf[s])
    assert np.array_equal(res[0][5], res[1][5])  # replicated multiplier, bitwise equal on both ranks

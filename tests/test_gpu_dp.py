"""Data parallel on the GPU kernels: 2 ranks (gloo, both on cuda:0 — the
driver's boxes have one GPU) each run the real training step on their shard
of the batch; the bucketed all-reduce of the parameter flows (per-layer
ranges started at the backward pass's flow events, then the input pmfs and
the zero tile) and the replicated EM must reproduce the one-process step —
the reference's threaded == serial check (tests/test_train.py:95-103) on the
device path.  NCCL needs one GPU per rank and is exercised by bench.py under
torchrun on multi-GPU nodes."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=30, hidden_dim=64,
                                       num_categories=8, seed=4))
    c = compile_circuit(g, CompileConfig(block_size=32))
    rng = np.random.default_rng(7)
    xs = [rng.integers(0, 8, size=(200, 30)) for _ in range(2)]
    data = rng.integers(0, 8, size=(450, 30))
    return c, xs, data


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2406_00766_b200.runtime.step import TrainStep
    from paper_2406_00766_b200.train import TrainConfig, shard_span, train
    c, xs, data = _case()
    theta0 = c.theta.copy()
    lo, hi = shard_span(200, rank, world)
    ts = TrainStep(c, hi - lo, pseudocount=1e-3, step_size=0.1, graph=False,
                   allreduce=lambda t: dist.all_reduce(t))
    assert ts._buckets is not None and len(ts._buckets) > 2  # per-layer buckets
    lls = []
    for x in xs:
        lls.append(float(ts.run(torch.from_numpy(x[lo:hi].astype(np.int32)).cuda()).item()))
    th_step = ts.plan.theta.double().cpu().numpy()
    from paper_2406_00766_b200.runtime.em import apply_theta
    apply_theta(c, theta0)
    res = train(c, data, TrainConfig(epochs=1, batch_size=128, mode="mini", step_size=0.05,
                                     pseudocount=1e-3, seed=1))
    out[rank] = (th_step, lls, c.theta.copy(), res.epoch_log_likelihood)
    dist.destroy_process_group()


def test_two_rank_gpu_steps_match_single_process():
    import torch
    import torch.multiprocessing as mp
    from paper_2406_00766_b200.runtime.em import apply_theta
    from paper_2406_00766_b200.runtime.step import TrainStep
    from paper_2406_00766_b200.train import TrainConfig, train
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    c, xs, data = _case()
    theta0 = c.theta.copy()
    ts = TrainStep(c, 200, pseudocount=1e-3, step_size=0.1, graph=False)
    lls = [float(ts.run(torch.from_numpy(x.astype(np.int32)).cuda()).item()) for x in xs]
    want = ts.plan.theta.double().cpu().numpy()
    apply_theta(c, theta0)
    res = train(c, data, TrainConfig(epochs=1, batch_size=128, mode="mini", step_size=0.05,
                                     pseudocount=1e-3, seed=1))
    want_train = c.theta.copy()
    (t0, l0, tr0, e0), (t1, l1, tr1, e1) = out[0], out[1]
    np.testing.assert_array_equal(t0, t1)  # replicated EM: bitwise identical ranks
    np.testing.assert_array_equal(tr0, tr1)
    assert l0 == l1
    np.testing.assert_allclose(l0, lls, rtol=1e-6)
    nz = np.abs(want) > 1e-7
    assert np.max(np.abs(t0[nz] - want[nz]) / np.abs(want[nz])) < 1e-5
    nz = np.abs(want_train) > 1e-7
    assert np.max(np.abs(tr0[nz] - want_train[nz]) / np.abs(want_train[nz])) < 1e-5
    np.testing.assert_allclose(e0, res.epoch_log_likelihood, rtol=1e-6)

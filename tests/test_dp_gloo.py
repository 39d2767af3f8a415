"""Data-parallel coordination on CPU: world_size 2 over gloo.

Exercises the exact helpers ``train()`` and ``bench.py`` use on GPUs —
``shard_span`` (the reference's ``_chunk_ranges`` split, train.py:78-81) and
``allreduce_accumulators`` (sum of f_params[:theta_size] and the log-
likelihood) — with the float64 oracle as the per-rank compute.  The merged
EM step must equal the single-process step (the reference's threaded ==
serial check, tests/test_train.py:95-103).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    g = S.build_hclt(S.StructureConfig(kind="hclt", num_vars=10, hidden_dim=8,
                                       num_categories=5, seed=2))
    c = compile_circuit(g, CompileConfig(block_size=8))
    x = np.random.default_rng(3).integers(0, 5, size=(37, 10))
    return c, x


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2406_00766_b200.train import allreduce_accumulators, shard_span
    c, x = _case()
    lo, hi = shard_span(x.shape[0], rank, world)
    lr, bufs = oracle.forward(c, x[lo:hi])
    oracle.backward(c, bufs)
    fp = torch.from_numpy(bufs.f_params.copy())
    ll = torch.tensor(float(lr.sum()), dtype=torch.float64)
    allreduce_accumulators(fp, ll, c.theta_size)
    theta = oracle.em_step_mini(c.theta, oracle.em_step_full(c, fp.numpy(), pseudocount=1e-6),
                                0.01)
    out[rank] = (theta, float(ll))
    dist.destroy_process_group()


def test_shard_span_covers_batch():
    from paper_2406_00766_b200.train import shard_span
    for n in (0, 1, 5, 37, 512):
        for world in (1, 2, 3, 8):
            spans = [shard_span(n, r, world) for r in range(world)]
            cover = [i for a, b in spans for i in range(a, b)]
            assert cover == list(range(n))


def test_two_rank_em_step_matches_single_process():
    import oracle
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    c, x = _case()
    lr, bufs = oracle.forward(c, x)
    oracle.backward(c, bufs)
    want = oracle.em_step_mini(c.theta,
                               oracle.em_step_full(c, bufs.f_params, pseudocount=1e-6), 0.01)
    t0, ll0 = out[0]
    t1, ll1 = out[1]
    np.testing.assert_array_equal(t0, t1)  # replicated EM stays bitwise identical
    np.testing.assert_allclose(t0, want, rtol=1e-12, atol=1e-15)
    assert ll0 == ll1
    np.testing.assert_allclose(ll0, float(lr.sum()), rtol=1e-12)

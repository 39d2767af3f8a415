"""Benchmark: samples/s of forward + backward + mini-batch EM on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload hclt256|hclt16|hmm4096|...]

One "step" = one pass of the hot path over one synthetic batch: input
gathers, product gather-adds, tcgen05 sum-layer contractions, parameter and
child flows, flow pushes, input flows, replica reduction, all-reduce of the
parameter flows (N > 1) and the fused mini-batch EM update (alpha 0.01,
pseudocount 1e-6) — the reference's ``train()`` inner loop
(``pcirc/train.py:128-142``).

``value``: inputs resident in HBM before the timed region, the step replayed
as a CUDA graph.  ``e2e``: one timed 60,000-sample epoch through the drop-in
``train()`` from a host (numpy) dataset — ceil(60000 / B) steps including the
tail batch, the per-epoch shuffle, host-side gathers and validation, every
batch copied host -> device (streamed behind the compute) and the epoch
log-likelihood read back; ``config.sec_per_epoch`` is that measured epoch.
Per-kernel-class times come from CUDA events recorded live on the launching
stream in a separate profiled pass.  Each class is reported against its
roofline: HBM GB/s from its algorithmic bytes, and for the sum contractions
also tensor TFLOP/s from its useful flops (2 x sum edges x B) against the
measured bf16 peak; ``roofline`` is the dominant class on the bound its
arithmetic intensity selects.  Every step's working set (GBs of values /
flows / parameters) exceeds the 126 MB L2, so no explicit flush is needed.
``--impl reference`` times the CPU oracle port of the reference on the host
cores instead (rank 0 only): forward + backward per sample and the EM pass
over the whole table timed separately and composed into a step of the
workload's batch size.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np

WORKLOADS = {
    "hclt256": dict(kind="hclt", num_vars=3072, hidden_dim=256, num_categories=256, block=32,
                    batch=512, desc="HCLT latent=256, 3072 vars (ImageNet32-shaped), 256 cats"),
    "hclt16": dict(kind="hclt", num_vars=784, hidden_dim=16, num_categories=256, block=16,
                   batch=512, desc="HCLT latent=16, 784 vars (MNIST-shaped), 256 cats"),
    "hclt64": dict(kind="hclt", num_vars=3072, hidden_dim=64, num_categories=256, block=32,
                   batch=512, desc="HCLT latent=64, 3072 vars, 256 cats (dev proxy)"),
    # deep trees: the same HCLT-256 on a breadth-first
    # spanning tree of the 32 x 32 x 3 pixel grid (a Chow-Liu-like tree of
    # neighbouring pixels: 64 levels) and on a path (3072 levels, the
    # latency-bound worst case)
    "hclt256_grid": dict(kind="hclt", num_vars=3072, hidden_dim=256, num_categories=256,
                         shape=(32, 32, 3), tree="grid", block=32, batch=512,
                         desc="HCLT latent=256 on a pixel-grid BFS tree (depth 64), 3072 vars"),
    "hclt256_chain": dict(kind="hclt", num_vars=3072, hidden_dim=256, num_categories=256,
                          tree="chain", block=32, batch=512,
                          desc="HCLT latent=256 on a path (depth 3072), 3072 vars"),
    "hmm4096": dict(kind="hmm", seq_len=32, hidden_dim=4096, vocab_size=50257, block=32,
                    batch=256, desc="HMM hidden=4096, vocab 50257, seq len 32"),
    # PyJuice PD (elementwise products per cut) on ImageNet32 (32 x 32 x 3):
    # cuts every 8 pixels, halving below; 213 M sum edges
    "pd256": dict(kind="pd", shape=(32, 32, 3), split_interval=8, hidden_dim=256,
                  num_categories=256, elementwise=True, block=32, batch=512,
                  desc="PD (PyJuice, elementwise cuts every 8 px) latent=256, 32x32x3, "
                       "256 cats"),
    # RAT-SPN on MNIST (784 vars): depth 7, 32 repetitions, 32 sums per region,
    # 32 factorised input components per leaf region; 137 M sum edges
    "ratspn": dict(kind="ratspn", num_vars=784, depth=7, hidden_dim=32,
                   num_input_components=32, num_repetitions=32, num_categories=256, block=32,
                   batch=1024, desc="RAT-SPN depth 7, 32 repetitions, 32 sums / 32 inputs per "
                                    "region, 784 vars, 256 cats"),
}
EPOCH = 60000
STEP_SIZE = 0.01
PSEUDOCOUNT = 1e-6


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def build_circuit(w):
    """Generate + compile the workload circuit.  ``PCB_CIRCUIT_CACHE=<dir>``
    pickles the compiled IR so repeated runs on one box skip the compile."""
    cache = os.environ.get("PCB_CIRCUIT_CACHE")
    if cache:
        import pickle
        key = "_".join(f"{k}{v}" for k, v in sorted(w.items()) if k != "desc")
        path = Path(cache) / f"{key}.pkl"
        if path.exists():
            with open(path, "rb") as f:
                return pickle.load(f)
        c = _build_circuit(w)
        path.parent.mkdir(parents=True, exist_ok=True)
        with open(path, "wb") as f:
            pickle.dump(c, f, protocol=5)
        return c
    return _build_circuit(w)


HOST_BUILD: dict = {}  # last _build_circuit's host timings (bench line: config.host_build)


def _build_circuit(w):
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, _native, compile_circuit
    keys = ("kind", "num_vars", "hidden_dim", "num_categories", "seq_len", "vocab_size",
            "shape", "split_interval", "elementwise", "depth", "num_input_components",
            "num_repetitions", "tree")
    cfg = S.StructureConfig(seed=0, tied=True, **{k: w[k] for k in keys if k in w})
    t0 = time.perf_counter()
    g = S.build_structure(cfg)
    t1 = time.perf_counter()
    c = compile_circuit(g, CompileConfig(block_size=w["block"]), validate=False)
    t2 = time.perf_counter()
    HOST_BUILD.clear()
    HOST_BUILD.update(structure_s=round(t1 - t0, 2), compile_s=round(t2 - t1, 2),
                      compiler="native" if _native.lib() is not None else "numpy",
                      host_threads=os.cpu_count())
    return c


def synthetic_batches(c, w, B, count, seed):
    """Uniform categories, ``default_rng(1)``-derived."""
    rng = np.random.default_rng([1, seed])
    cats = np.asarray(c.var_categories)
    return [rng.integers(0, cats[None, :], size=(B, c.num_vars)).astype(np.int32)
            for _ in range(count)]


def fused_em_bytes(c, info, B, sms=148):
    """(edges of the layers whose EM runs in the parameter-flow epilogue at
    batch B, staged input pmf entries updated in the input-flow pass): the
    plan's em-fusable layers whose parameter flows are unsplit (the C side's
    pf_kslices == 1 for every group)."""
    from paper_2406_00766_b200.runtime.plan import tc_super_rows
    e_f = 0
    for li in info.get("em_fused_layer_ids", []):
        L = c.layers[li]
        ok, e = True, 0
        for g in L.fwd_groups:
            offs, _ = tc_super_rows(g.prod_ids, L.k_m, min_count=0)
            cg = -(-int(g.prod_ids.shape[1]) * int(L.k_n) // 256)
            base = (offs.size - 1) * cg * 2
            ks = max(1, min(-(-2 * sms // max(base, 1)), (-(-B // 32)) // 2))
            ok = ok and ks == 1
            e += int((np.asarray(g.param_ids) != 0).sum()) * int(L.k_m) * int(L.k_n)
        e_f += e if ok else 0
    n_pmf = 0
    if info.get("input_inline_em"):
        n_pmf = sum(int(ch.param_ids.size) * int(ch.num_categories) for ch in c.input_layer)
    return e_f, n_pmf


def _layer_counts(c, L):
    n_sum = int(L.report.num_sums)
    n_prod = int(L.report.num_prods)
    F = sum(int(ev.children.size) for ev in L.prod_evals)
    E = int(L.edge_sums.size)
    # tile work the contraction executes (real (row, column) tile pairs)
    E_pad = sum(int((np.asarray(g.param_ids) != 0).sum()) for g in L.fwd_groups) * L.k_m * L.k_n
    return n_sum, n_prod, F, E, E_pad


def class_model(c, B, info=None):
    """Per kernel class of the lean training step: minimal fp32 HBM bytes per
    step and, for the sum contractions, useful flops per step
    (2 x sum edges x B, one multiply-add per edge and sample) and the
    executed bf16 MMA flops (3 MMAs per 16-wide K step: hi*hi + hi*lo + lo*hi,
    over the real tiles).  Products stay resident (evaluated once), the first
    layer's products alias their inputs when the plan allows it, the fused
    push moves each pushed product flow to its children once; each tied pmf
    is read once.  Only the layers a class actually runs are counted (sum
    layers of block size 16 / 32 on tensor cores, the rest SIMT)."""
    from paper_2406_00766_b200.runtime.plan import tc_layer
    info = info or {}
    skip = 1 if info.get("leaf_alias") else 0  # aliased first layer: no product pass / push
    n_in = sum(int(ch.node_ids.size) for ch in c.input_layer)
    pmf = set()
    for ch in c.input_layer:
        pmf.update((int(p), int(ch.num_categories)) for p in np.unique(ch.param_ids))
    n_pmf = sum(k for _, k in pmf)
    m = {k: {"bytes": 0, "flops": 0, "mma_flops": 0} for k in
         ("input_fwd", "prod_eval", "sum_fwd_tc", "sum_fwd_simt", "param_flow", "child_flow",
          "accum_push", "input_flow", "em")}
    m["input_fwd"]["bytes"] = B * 4 * (c.num_vars + n_in) + 4 * n_pmf
    m["input_flow"]["bytes"] = B * 4 * (n_in + c.num_vars) + 8 * n_pmf
    m["em"]["bytes"] = 20 * c.theta_size
    # parameter tiles: a tile shared by several layers (tied HMM transitions)
    # is read (and its flows accumulated) once per step at minimum — charge
    # each unique tile to the first layer that uses it
    seen = set()
    for li, L in enumerate(c.layers):
        n_sum, n_prod, F, E, E_pad = _layer_counts(c, L)
        tc = tc_layer(L) and L.k_m in (16, 32, 64) and L.k_n in (16, 32)
        fwd = "sum_fwd_tc" if tc else "sum_fwd_simt"
        if li >= skip:
            m["prod_eval"]["bytes"] += B * 4 * (F + n_prod)
            m["accum_push"]["bytes"] += B * 4 * (n_prod + F + n_sum)
        tiles = set()
        for g in L.fwd_groups:
            pid = np.asarray(g.param_ids)
            tiles.update(np.unique(pid[pid != 0]).tolist())
        new = tiles - seen
        seen |= tiles
        E_u = E * len(new) // max(len(tiles), 1)  # edges in tiles not yet charged
        m[fwd]["bytes"] += B * 4 * (n_prod + n_sum) + 4 * E_u
        # ratio rows + product offsets; theta read + flow write per unique edge
        m["param_flow"]["bytes"] += B * 4 * (n_sum + n_prod) + 8 * E_u
        # ratio rows + product offsets + product-flow rows; theta (bf16 planes)
        m["child_flow"]["bytes"] += B * 4 * (n_sum + 2 * n_prod) + 4 * E_u
        for k in (fwd, "param_flow", "child_flow"):
            m[k]["flops"] += 2 * E * B
            if tc:
                m[k]["mma_flops"] += 3 * 2 * E_pad * B
    return m


def algorithmic_bytes(c, B, info=None):
    return {k: v["bytes"] for k, v in class_model(c, B, info).items()}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _nvml(self):
        """In-process NVML reads (every 10 ms), else None."""
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                N.nvmlDeviceGetCurrentClocksThrottleReasons
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)

            def read():
                r = get_reasons(h)
                act = lambda bit: "Active" if r & bit else "Not Active"  # noqa: E731
                return [str(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)), str(mx), hex(r),
                        act(0x8), act(0x40), act(0x20), act(0x4)]
            read()
            return read
        except Exception:
            return None

    def _sample(self):
        try:
            if self._read is not None:
                self.rows.append(self._read())
        except Exception:
            pass

    def _run(self):
        read = self._read
        while not self._stop.is_set():
            try:
                if read is not None:
                    self.rows.append(read())
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout.strip()
                    if out:
                        self.rows.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.01 if read is not None else 0.2)

    def __enter__(self):
        self._read = self._nvml()  # initialised before the timed region starts
        self._sample()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._sample()  # the state at the end of the device work
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6554.9), d.get("bf16_tflops_sustained", 1420.9), "measured"
    return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------- CPU oracle
def cpu_step_parts(c, w, B_cpu, seed=7, em=True):
    """Oracle (float64 numpy port of the reference) on B_cpu samples: seconds
    of forward + backward, and of the EM pass (em_step_full + em_step_mini
    over the whole table, independent of the batch size; 0 when em=False)."""
    import oracle
    x = synthetic_batches(c, w, B_cpu, 1, seed)[0].astype(np.int64)
    theta = c.theta.copy()
    t0 = time.perf_counter()
    _, bufs = oracle.forward(c, x, theta=theta)
    oracle.backward(c, bufs, theta=theta)
    t1 = time.perf_counter()
    if not em:
        return t1 - t0, 0.0
    new = oracle.em_step_full(c, bufs.f_params, theta=theta, pseudocount=PSEUDOCOUNT)
    if new is not None:
        theta = oracle.em_step_mini(theta, new, STEP_SIZE)
    return t1 - t0, time.perf_counter() - t1


def cpu_sample_size(w):
    """Samples per timed CPU forward + backward: the full batch where it fits
    in seconds, else a bounded sample."""
    if w["kind"] == "hmm":
        return 4
    return {16: 512, 64: 64}.get(w["hidden_dim"], 32)


def composed(w, B_cpu, t_fb, t_em):
    """A step of the workload's batch B composed from the measured parts:
    B / B_cpu x forward+backward(B_cpu) + EM (the reference's per-sample cost
    is linear in B; its EM pass is one full-table pass per step)."""
    B = w["batch"]
    t = B / B_cpu * t_fb + t_em
    return B / t, t, (f"step(B={B}) = {B}/{B_cpu} x {t_fb:.2f} s (fwd+bwd on {B_cpu} samples) "
                      f"+ {t_em:.2f} s (EM over theta) = {t:.1f} s")


def run_reference(args, w):
    """--impl reference: the oracle port timed on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    c = build_circuit(w)
    # per step: forward + backward on a bounded sample (a sixteenth of the
    # baseline sample keeps K + W steps within minutes); the batch-independent
    # EM pass over the whole table is timed once after the steps
    Bc = max(1, cpu_sample_size(w) // 16)
    for i in range(args.warmup):
        cpu_step_parts(c, w, Bc, seed=100 + i, em=False)
    fb = 0.0
    for i in range(args.steps):
        fb += cpu_step_parts(c, w, Bc, seed=i, em=False)[0]
    em = cpu_step_parts(c, w, Bc, seed=99)[1]
    v, t, formula = composed(w, Bc, fb / args.steps, em)
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": "samples/sec fwd+bwd+EM", "value": v,
        "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * t, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "desc": w["desc"], "batch_per_step": w["batch"],
                   "sampled_batch": Bc, "composition": formula, "sec_per_epoch": EPOCH / v},
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "port",
                         "sample": f"per step: forward+backward on {Bc} samples of the "
                                   f"{args.workload} workload + the EM pass over the full "
                                   f"theta, composed to batch {w['batch']}: {formula}"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def secondary(name, args, dev, world, rank, graphed):
    """Another BASELINE config measured in the same run (device-resident
    steps and a 60k-sample train() epoch from host data), reported under
    ``secondary`` of the JSON line."""
    import torch
    import torch.distributed as dist
    from paper_2406_00766_b200.train import TrainConfig, cached_step, shard_span, train
    w = WORKLOADS[name]
    t0 = time.time()
    c = build_circuit(w)
    compile_s = time.time() - t0
    G = w["batch"]
    lo, hi = shard_span(G, rank, world)
    B = hi - lo
    xs = [torch.from_numpy(h).to(dev) for h in synthetic_batches(c, w, B, 2, seed=rank)]
    ts = cached_step(c, B, pseudocount=PSEUDOCOUNT, step_size=STEP_SIZE, device=dev,
                     graph=graphed)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        ts.run(xs[i % 2])
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        ts.run(xs[i % 2])
    e1.record()
    barrier()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / args.steps
    data = synthetic_batches(c, w, EPOCH, 1, seed=11)[0]
    cfg = TrainConfig(epochs=1, batch_size=G, mode="mini", step_size=STEP_SIZE,
                      pseudocount=PSEUDOCOUNT, seed=0)
    train(c, data[: 2 * G + EPOCH % G], cfg, device=dev, graph=graphed)
    barrier()
    res = train(c, data, cfg, device=dev, graph=graphed)
    t = torch.tensor([res.epoch_seconds[0]], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ep = float(t.item())
    return {"desc": w["desc"], "edges": c.num_edges, "theta_size": c.theta_size,
            "global_batch": G, "value": G / (ms / 1000.0), "unit": "samples/s",
            "ms_per_step": ms, "e2e": {"value": EPOCH / ep, "unit": "samples/s",
                                       "sec_per_epoch": ep}, "compile_s": compile_s}


def run_ours(args, w):
    import torch
    import torch.distributed as dist
    from paper_2406_00766_b200.runtime import _lib
    from paper_2406_00766_b200.train import cached_step, shard_span

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; PCB_DIST_BACKEND=gloo (with ranks sharing a GPU)
    # exercises the multi-rank path where fewer GPUs than ranks exist
    backend = os.environ.get("PCB_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    t0 = time.time()
    c = build_circuit(w)
    host_build = dict(HOST_BUILD)
    log(f"[bench] compiled {args.workload}: {c.num_edges} edges, theta {c.theta_size} "
        f"in {time.time() - t0:.1f}s {host_build}")
    # strong scaling (north_star: the config's mini-batch is sharded across
    # the GPUs): global batch = the config's, this rank's contiguous span of
    # it (the reference's _chunk_ranges split); --scaling weak keeps the
    # per-GPU batch fixed instead
    G = w["batch"] * (world if args.scaling == "weak" else 1)
    lo, hi = shard_span(G, rank, world)
    B = hi - lo
    n_pool = 4
    host_batches = synthetic_batches(c, w, B, n_pool, seed=rank)
    dev_batches = [torch.from_numpy(h).to(dev) for h in host_batches]
    ll_acc = torch.zeros((), dtype=torch.float64, device=dev)

    # the training step as a CUDA graph (the batch is copied into a static
    # input buffer, every kernel replays without host launches); on N > 1 the
    # bucketed NCCL all-reduce of the parameter flows is captured with it.
    # The same cached step (buffers, graph) serves train() below.
    graphed = not args.no_graph and (world == 1 or backend == "nccl")
    t0 = time.perf_counter()
    ts = cached_step(c, B, pseudocount=PSEUDOCOUNT, step_size=STEP_SIZE, device=dev,
                     graph=graphed)
    host_build["plan_and_upload_s"] = round(time.perf_counter() - t0, 2)
    plan = ts.plan
    run = ts.run

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (also builds every lazily created kernel attribute)
    for i in range(args.warmup):
        run(dev_batches[i % n_pool])
    barrier()

    # ---- device-resident timed region
    launches0 = _lib.load().pcb_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier()
        ev0.record()
        for i in range(args.steps):
            ll_acc += run(dev_batches[i % n_pool])
        ev1.record()
        torch.cuda.synchronize()  # the sampler covers the device work, not just the enqueue
        barrier()
    launches = _lib.load().pcb_launch_count() - launches0
    if graphed:  # replays launch the captured kernels without host calls
        launches = ts.launches_per_step * args.steps
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    value = G * args.steps / (ms / 1000.0)

    # ---- profiled pass: live per-kernel-class CUDA-event times
    prof_steps = max(1, min(3, args.steps))
    _lib.profile_enable(True)
    _lib.profile_read()
    # eager: the class timers are host-side event pairs; the side-stream
    # overlap is switched off so each class is timed on its own
    ts.serial = True
    for i in range(prof_steps):
        ts._eager(dev_batches[i % n_pool])
    torch.cuda.synchronize()
    ts.serial = False
    prof = _lib.profile_read()
    _lib.profile_enable(False)

    # ---- end to end: one 60k-sample epoch through train() from host data
    from paper_2406_00766_b200.train import TrainConfig, train
    n_ep = EPOCH
    data = synthetic_batches(c, w, n_ep, 1, seed=11)[0]  # identical on every rank

    def epoch(mode, gb):
        """One timed epoch through train() (after a short untimed call that
        builds its steps: full batches and the tail)."""
        tcfg = dict(batch_size=gb, mode=mode, step_size=STEP_SIZE, pseudocount=PSEUDOCOUNT,
                    seed=0)
        train(c, data[: 2 * gb + n_ep % gb], TrainConfig(epochs=1, **tcfg), device=dev,
              graph=graphed)
        barrier()
        res = train(c, data, TrainConfig(epochs=1, **tcfg), device=dev, graph=graphed)
        t = torch.tensor([res.epoch_seconds[0]], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), -(-n_ep // gb)

    ep_s, n_steps_ep = epoch("mini", G)
    e2e_value = n_ep / ep_s
    # full-batch EM (train.py:130-146, the reference's default mode): one
    # all-reduce and EM pass per epoch, so each GPU runs a full config batch
    # per step at any N
    fb_s, fb_steps = epoch("full", w["batch"] * world)
    full_batch = {"value": n_ep / fb_s, "unit": "samples/s", "sec_per_epoch": fb_s,
                  "steps": fb_steps, "batch_per_gpu": w["batch"], "global_batch":
                  w["batch"] * world, "how": "one 60k-sample epoch through train(mode='full')"
                                             " from host data, one EM per epoch"}

    # other BASELINE configs in the same run (every rank takes part)
    sec = {}
    for name in [n for n in args.secondary.split(",") if n and n != args.workload]:
        try:
            sec[name] = secondary(name, args, dev, world, rank, graphed)
        except Exception as e:  # a secondary never sinks the headline line
            sec[name] = {"error": f"{type(e).__name__}: {e}"}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    hbm, tflops, peak_src = measured_peaks()
    model = class_model(c, B, ts.plan.info)
    # one-process steps fold EM into the input-flow and parameter-flow passes
    # (DESIGN §3a): the EM class then covers only the small layers' groups, and
    # the per-class minimal bytes above (unfused) no longer describe it
    inline_em = world == 1
    if inline_em:
        model["em"]["bytes"] = None
        # the fused EM's extra minimal bytes: theta write + four bf16 planes
        # instead of the flow write per edge of the layers whose parameter
        # flows run unsplit, theta read + write instead of the flow write per
        # staged input pmf entry
        e_f, n_pmf = fused_em_bytes(c, ts.plan.info, B)
        model["param_flow"]["bytes"] += 8 * e_f
        model["input_flow"]["bytes"] += 4 * n_pmf
    classes = {k: v for k, v in prof.items() if v[0] > 0}
    total_prof = sum(v[0] for v in classes.values())
    ridge = tflops * 1e12 / (hbm * 1e9)  # flop / byte where the two roofs meet

    def figures(k, ms):
        sec = ms / 1000.0
        mk = model.get(k, {})
        by, fl, mm = mk.get("bytes"), mk.get("flops", 0), mk.get("mma_flops", 0)
        f = {"ms_per_step": ms}
        if by:
            f["gbs"] = by / sec / 1e9
            f["hbm_frac"] = f["gbs"] / hbm
        if fl:
            f["tflops"] = fl / sec / 1e12
            f["tensor_frac"] = f["tflops"] / tflops
            f["mma_tflops_executed"] = mm / sec / 1e12 if mm else None
            f["flop_per_byte"] = fl / by if by else None
        return f

    breakdown = {}
    for k, v in classes.items():
        breakdown[k] = figures(k, v[0] / prof_steps)
        breakdown[k]["launches_per_step"] = v[2] / prof_steps
    dom = max(classes, key=lambda k: classes[k][0])
    dom_ms, dom_scopes, dom_launches = classes[dom]
    per_step_ms = dom_ms / prof_steps
    fd = breakdown[dom]
    mk = model.get(dom, {})
    ai = (mk.get("flops", 0) / mk["bytes"]) if mk.get("bytes") else None
    tensor_bound = bool(ai) and ai >= ridge
    traffic = None
    tr_file = ROOT / "profiles" / f"traffic_{args.workload}.json"
    if tr_file.exists():
        traffic = json.loads(tr_file.read_text()).get(dom)
    if tensor_bound:
        achieved, peak, unit = fd["tflops"], tflops, "TFLOP/s"
    else:
        achieved, peak, unit = fd.get("gbs"), hbm, "GB/s"
    roofline = {"bound": "tensor" if tensor_bound else "hbm", "kernel": dom,
                "achieved": achieved, "peak": peak, "unit": unit,
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "peak_source": peak_src + (" (bf16 sustained)" if tensor_bound else " (copy)"),
                "algorithmic_bytes_per_step": mk.get("bytes"),
                "useful_flops_per_step": mk.get("flops") or None,
                "flop_per_byte": ai, "ridge_flop_per_byte": ridge,
                "hbm_frac": fd.get("hbm_frac"), "tensor_frac": fd.get("tensor_frac"),
                "kernel_ms_per_step": per_step_ms,
                "launches_per_step": dom_launches / prof_steps,
                "share_of_step": dom_ms / total_prof if total_prof else None}

    cpu = None
    if world == 1 and not args.no_cpu:
        Bc = cpu_sample_size(w)
        t_fb, t_em = cpu_step_parts(c, w, Bc)
        v, t, formula = composed(w, Bc, t_fb, t_em)
        cpu = {"value": v, "unit": "samples/s", "cores": os.cpu_count(), "kind": "port",
               "sample": f"forward+backward on {Bc} samples of {args.workload} + the EM pass "
                         f"over the full theta, composed to batch {B} (numpy float64, BLAS "
                         f"threads = host cores): {formula}"}
    line = {
        "metric": "samples/sec fwd+bwd+EM", "value": value, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": args.workload, "desc": w["desc"], "batch_per_gpu": B,
                   "global_batch": G, "block_size": w["block"],
                   "em": f"mini-batch, step {STEP_SIZE}, pseudocount {PSEUDOCOUNT}",
                   "edges": c.num_edges, "theta_size": c.theta_size,
                   "sec_per_epoch": ep_s,
                   "sec_per_epoch_note": f"measured: one {n_ep}-sample epoch through train() "
                                         f"({n_steps_ep} steps incl. the tail batch) from host "
                                         "data",
                   "l2": "working set >> 126 MB L2 (no flush)",
                   "parallelism": f"dp{world}", "cuda_graph": graphed,
                   "em_in_backward": inline_em,
                   "host_build": host_build or "loaded from PCB_CIRCUIT_CACHE"},
        "e2e": {"value": e2e_value, "unit": "samples/s",
                "h2d_bytes_per_step": B * c.num_vars * 4,
                "d2h_bytes_per_step": 8,
                "how": f"train(): {n_ep}-sample epoch, host numpy int32 dataset, shuffle + "
                       "per-batch gather / validation on a loader thread, pinned H2D copies "
                       "streamed behind the compute"},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "kernels": breakdown,
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
        "full_batch_em": full_batch,
    }
    if sec:
        line["secondary"] = sec
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="hclt256", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every kernel eagerly")
    ap.add_argument("--secondary", default="hclt16",
                    help="comma-separated other workloads measured in the same run "
                         "(value + train() epoch) under 'secondary', e.g. hclt16,pd256,ratspn")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's batch sharded over the GPUs (north_star); "
                         "weak: the config's batch per GPU")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()

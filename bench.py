#!/usr/bin/env python3
"""bench.py -- connection evaluations per second of the ASNN activation sweep.

Metric (BASELINE.json): edges/sec (connection evals/s) + HBM GB/s vs roofline
at 1/2/4/8 B200 vs host CPU.  Headline workload: config 4, a large power-law
ASNN (~10M nodes, ~500M edges) with a batch of 64 input vectors sharded over
the GPUs.  One step = one full activation sweep (sensors,
every dependency level, output gather) of the whole batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
  python bench.py --impl reference ...      # the reference's CPU evaluator

Multi-GPU: torchrun, one rank per GPU, each rank holds the full CSR and its
64/N batch columns (no per-level traffic); outputs are all-gathered with NCCL.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "connection evals/s (edges x vectors per second), full activation sweep"
DATA = "synthetic (seeded generator, DESIGN.md corpora)"

CONFIGS = {
    # name: (description, builder kwargs, batch)
    "c1": ("small random ASNN (1k nodes, 10k connections), single input vector", 1),
    "c2": ("pruned-MLP sparse network (100k nodes, ~5M edges, 90% sparsity), batch 1024", 1024),
    "c3": ("deep narrow NEAT-style DAG (50k nodes, 2000 levels), batch 256", 256),
    "c4": ("large random power-law ASNN (10M nodes, ~500M edges), batch 64", 64),
    "c5": ("NEAT population: 10k networks x 200 nodes, 128 inputs each", 128),
}


def make_network(cfg: str, scale: float = 1.0):
    import paper_2005_04347_b200 as A
    if cfg == "c1":
        return [A.generate(A.GenSpec(16, 4, 980, 10000, 10, -1.0, 1.0, 1))]
    if cfg == "c2":
        return [A.generate_mlp(200, 500, 0.1, 2)]
    if cfg == "c3":
        return [A.generate(A.GenSpec(16, 4, 49980, 500000, 2000, -1.0, 1.0, 3))]
    if cfg == "c4":
        n = int(10_000_000 * scale)
        return [A.generate_powerlaw(n, 100, 1024, 1024, int(500_000_000 * scale), 2.1, 4)]
    if cfg == "c5":
        rng = A.SplitMix64(5)
        count = int(10_000 * scale)
        return [A.generate(A.GenSpec(8, 4, 188, 1000, 8, -1.0, 1.0, rng.next())) for _ in range(count)]
    raise ValueError(cfg)


def band_starts(cfg: str, net) -> np.ndarray:
    """Level boundaries of the banded generators (configs 2 and 4): every
    non-input node has a mandatory predecessor in the previous band and all
    sources in earlier bands, so its level is its band and positions in
    (level, id) order are the ids themselves (netgen.cpp)."""
    N = len(net.nodes)
    if cfg == "c2":
        return np.arange(0, N + 1, 500, dtype=np.uint32)
    n_in, n_out, bands = len(net.inputs), len(net.outputs), 100
    hidden = N - n_in - n_out
    base, rem = divmod(hidden, bands - 2)
    sizes = [n_in] + [base + (1 if b < rem else 0) for b in range(bands - 2)] + [n_out]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)


def host_layout_banded(cfg: str, net) -> dict:
    """Flattened layout of a banded generator network, straight from the
    generator's target-major edge list (sources already ascending)."""
    N = len(net.nodes)
    counts = np.bincount(net.target, minlength=N).astype(np.uint64)
    row_ptr = np.zeros(N + 1, np.uint64)
    np.cumsum(counts, out=row_ptr[1:])
    starts = band_starts(cfg, net)
    return dict(total_layers=len(starts) - 1, layer_offsets=starts, node_ids=net.nodes,
                row_ptr=row_ptr, in_nodes=net.source, in_weights=net.weight,
                input_order=net.inputs, id_bound=N, dropped_connections=0)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def profiled_traffic(cfg):
    """DRAM bytes per sweep from the committed ncu launch list (same unit as
    alg_bytes_per_step), or None when this config was not captured."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        e = json.loads(p.read_text()).get(cfg)
        if e:
            return e["dram_bytes_per_step"]
    return None


def make_network_ref(cfg: str, scale: float = 1.0):
    """The same corpora as make_network without the engine, for the
    reference arm: configs 1, 3 and 5 from the reference's own generate()
    (netgen.cpp:71-157 in oracle/_ref, byte-identical to the engine's
    restatement -- tests/test_corpus.py), configs 2 and 4 from the bench
    generators compiled out of csrc/netgen.cpp into oracle/libcorpus.so.
    Returns NetArrays (plain arrays) or, for configs 1/3/5, RefNet handles."""
    from oracle.bind import Corpus, Ref, SplitMix64
    if cfg == "c2":
        return [Corpus().mlp(200, 500, 0.1, 2)]
    if cfg == "c4":
        n = int(10_000_000 * scale)
        return [Corpus().powerlaw(n, 100, 1024, 1024, int(500_000_000 * scale), 2.1, 4)]

    class Spec:
        def __init__(self, i, o, h, c, d, seed):
            self.input_count, self.output_count, self.hidden_count = i, o, h
            self.connection_count, self.target_depth, self.seed = c, d, seed
            self.weight_min, self.weight_max = -1.0, 1.0
    ref = Ref()
    if cfg == "c1":
        return [ref.generate(Spec(16, 4, 980, 10000, 10, 1))]
    if cfg == "c3":
        return [ref.generate(Spec(16, 4, 49980, 500000, 2000, 3))]
    if cfg == "c5":
        rng = SplitMix64(5)
        return [ref.generate(Spec(8, 4, 188, 1000, 8, rng.next())) for _ in range(int(10_000 * scale))]
    raise ValueError(cfg)


def net_counts(net):
    """(nodes, inputs, edges) of a network given as arrays or a RefNet handle."""
    if hasattr(net, "h"):
        L = net.L
        return L.ref_net_n_nodes(net.h), L.ref_net_n_inputs(net.h), L.ref_net_n_edges(net.h)
    return len(net.nodes), len(net.inputs), len(net.source)


def config_dict(cfg: str, nets, world: int) -> dict:
    """The workload description both arms print (identical keys and values)."""
    counts = [net_counts(n) for n in nets]
    B = CONFIGS[cfg][1]
    per_gpu = B if cfg == "c5" else -(-B // world)
    return {"workload": CONFIGS[cfg][0], "config": cfg,
            "edges": int(sum(c[2] for c in counts)), "nodes": int(sum(c[0] for c in counts)),
            "networks": len(nets), "batch": B, "batch_per_gpu": per_gpu,
            "parallelism": (f"population-sharded x{world}" if cfg == "c5" else
                            f"batch-sharded dp{world}"),
            "l2": "working set > 126 MB L2 (no flush)" if cfg in ("c2", "c4") else
                  "L2-resident working set; per-step state rewritten"}


class RefCPU:
    """The reference's own CPU evaluator (oracle/_ref: the unmodified reference
    compiled from its sources) prepared once on the same networks; each
    measurement times a bounded sample of input vectors of that workload.

    Modes (all the reference's unchanged code):
      "seq"     eval_sequential on ONE core, vector by vector (bench.cpp:82-83);
      "par"     eval_parallel with all host threads, vector by vector;
      "omp-seq" an OpenMP loop of eval_sequential over `threads` vectors.
    For C5 the sample is the first `max_nets` networks of the population (each
    with its own vectors).  `nets` are NetArrays / api.Network objects, or
    RefNet handles from the reference's own generator."""

    MODES = {"seq": 0, "par": 1, "omp-seq": 2}

    def __init__(self, nets, X_all, cfg, max_nets=64):
        from oracle.bind import Oracle, Ref, RefNet, available_ref
        self.kind = "reference" if available_ref() else "port"
        self.ref = Ref() if self.kind == "reference" else None
        self.oracle = None if self.ref else Oracle()
        # all host threads: torchrun exports OMP_NUM_THREADS=1 to every rank, so
        # ask the OS (affinity) rather than OpenMP's default
        host = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        self.threads = max(self.ref.L.ref_max_threads(), host or 1) if self.ref else 1
        self.items = []
        self.evaluated = 0
        self.repeated = 0
        for gi, net in enumerate(nets[:max_nets]):
            if isinstance(net, RefNet):
                h = net
                assert h.preprocess() == 0
            elif cfg in ("c2", "c4"):
                # reference preprocessing of C4 takes ~20 min: build its
                # LayeredLayout straight from the banded CSR instead -- the
                # identical layout (sha256 equal to the reference's own
                # flatten, tests/test_oracle_golden.py::test_banded_layout_is_reference_flatten)
                lay = host_layout_banded(cfg, net)
                h = self.ref.layout_from_csr(lay) if self.ref else lay
            elif self.ref:
                h = self.ref.network(net)
                assert h.preprocess() == 0
            else:
                h = self.oracle.layout(net)
            E = net_counts(net)[2]
            ev = self.ref.L.ref_layout_edge_count(h.h) if self.ref else len(h["in_nodes"])
            X = X_all[gi]
            if X.shape[0] < 64:
                # a one-vector workload (C1): time its vector repeated, one
                # reference call per vector as before, so the sample is not a
                # single 10-us measurement
                self.repeated = X.shape[0]
                X = np.ascontiguousarray(np.tile(X, (-(-256 // X.shape[0]), 1))[:256])
            self.items.append((h, E, X))
            self.evaluated += ev
        self.n_nets = len(self.items)

    def run(self, mode, n_vec):
        """(conn_evals, seconds) of n_vec vectors per sampled network."""
        ev, dt = 0, 0.0
        for h, E, X in self.items:
            Xs = X[:n_vec]
            if self.ref is None:
                t0 = time.perf_counter()
                self.oracle.eval_batch(h, Xs)
                t = time.perf_counter() - t0
            else:
                t, _ = h.eval_batch(Xs, mode=self.MODES[mode],
                                    workers=1 if mode == "seq" else self.threads)
            ev += E * len(Xs)
            dt += t
        return ev, dt

    def sample_mode(self, mode, budget_s):
        """Vectors one call at a time (several at once for omp-seq) until about
        budget_s seconds are spent: (conn_evals, seconds, vectors)."""
        ev = dt = 0.0
        n = 0
        n_max = self.items[0][2].shape[0]
        step = self.threads if mode == "omp-seq" else 1
        self.run(mode, min(step, n_max))            # untimed: first-touch, thread team
        while (n == 0 or dt < budget_s) and n < n_max:
            k = min(step, n_max - n) if mode != "omp-seq" else min(step, n_max)
            e, t = self.run(mode, k)
            ev, dt, n = ev + e, dt + t, n + k
            if mode == "omp-seq":
                break
        return ev, dt, n

    def measure(self, budget_s=20.0):
        """All three modes on a bounded sample (about budget_s/3 s each); the
        best one is the baseline, every mode is reported by name."""
        if self.ref is None:
            ev, dt = self.run("par", 1)
            return self.describe("port-seq", ev, dt, 1)
        # omp-seq runs one vector per thread: not a mode for a workload with
        # fewer vectors than threads (its repeats are not extra work to share)
        modes = ("seq", "par") if self.repeated else ("seq", "par", "omp-seq")
        res = {m: self.sample_mode(m, budget_s / len(modes)) for m in modes}
        mode = max(res, key=lambda k: res[k][0] / res[k][1])
        d = self.describe(mode, *res[mode])
        d["modes"] = {m: {"value": r[0] / r[1], "cores": 1 if m == "seq" else self.threads,
                          "vectors": r[2], "seconds": r[1]} for m, r in res.items()}
        return d

    def describe(self, mode, ev, dt, n_vec):
        rep = f" (its {self.repeated} input vector(s) repeated)" if self.repeated else ""
        return {"value": ev / dt, "unit": "conn_evals/s",
                "cores": 1 if mode in ("seq", "port-seq") else self.threads, "kind": self.kind,
                "mode": mode,
                "sample": f"{n_vec} vector(s) x {self.n_nets} network(s) of this workload{rep} in "
                          f"{dt:.4f}s ({mode})"}


def cpu_baseline(nets, X_all, cfg, budget_s=20.0):
    return RefCPU(nets, X_all, cfg).measure(budget_s)


def run_ours(args, cfg):
    """Our arm.  One process per GPU (torchrun for N > 1).  Every rank holds
    a full layout replica and sweeps its contiguous slice of the batch (C5:
    its contiguous slice of the population); a step is the sweep plus the
    all-gather of the declared outputs, which the engine enqueues on its own
    stream right after the sweep (NCCL, asnn_dev_allgather).  With
    ASNN_BENCH_ONE_GPU=1 every rank shares GPU 0 -- a functional check of the
    N > 1 path: NCCL cannot place two ranks on one device, so the gather then
    goes through torch.distributed (gloo) on the host, still inside the step."""
    import torch
    import paper_2005_04347_b200 as A
    from paper_2005_04347_b200.shard import batch_slice, population_shard

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    one_gpu = bool(os.environ.get("ASNN_BENCH_ONE_GPU"))
    if one_gpu:
        local = 0
    dist = None
    if world > 1:
        import torch.distributed as dist
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    t_setup = time.perf_counter()
    nets = make_network(cfg, args.scale)
    B_total = CONFIGS[cfg][1]
    rng = np.random.default_rng(12345)
    shards = args.shard_of or world
    if cfg == "c5":
        X = [rng.uniform(-2, 2, (B_total, len(n.inputs))).astype(np.float32) for n in nets]
        owned = [population_shard(len(nets), world, r) for r in range(world)]
        mine = owned[rank]
        shard = [nets[g] for g in mine]
        Xs = [X[g] for g in mine]
        B = B_total
        out_counts = [B * sum(len(nets[g].outputs) for g in o) for o in owned]
    else:
        shard = nets
        X_full = rng.uniform(-2, 2, (B_total, len(nets[0].inputs))).astype(np.float32)
        X = [X_full]
        # --shard-of G (development): one process measuring rank 0's slice of a
        # G-way split, i.e. the per-GPU workload of a G-GPU run
        slices = [batch_slice(B_total, shards, r) for r in range(world)]
        lo, hi = slices[rank]
        Xs = [X_full[lo:hi]]
        B = hi - lo
        out_counts = [(h - l) * len(nets[0].outputs) for l, h in slices]
    t_gen = time.perf_counter() - t_setup

    dev = A.Device.get(local)
    # one explicit stream shared by the engine, its gather and the timing events
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    dev.set_stream(stream.cuda_stream)
    gather = "none (one GPU)"
    engine_gather = False
    if dist is not None:
        if one_gpu:
            gather = "gloo on the host (one-GPU functional mode)"
        else:
            # the engine's own communicator; if it cannot be created the step
            # gathers through torch.distributed (NCCL) instead, and says so
            ok = 1
            try:
                uid = [A.comm_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                dev.comm_init(uid[0], world, rank)
            except Exception as e:  # pragma: no cover - multi-GPU boxes only
                print(f"[rank {rank}] engine NCCL communicator unavailable: {e}", file=sys.stderr)
                ok = 0
            flag = torch.tensor([ok], device=f"cuda:{local}")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            engine_gather = bool(flag.item())
            gather = ("nccl all-gather in the engine (asnn_dev_allgather)" if engine_gather else
                      "nccl all-gather through torch.distributed (engine communicator unavailable)")
    t0 = time.perf_counter()
    if cfg == "c5":
        dl = A.DeviceLayout.from_population(shard, device=local)
    elif args.prep == "upload" and cfg in ("c2", "c4"):
        d = host_layout_banded(cfg, shard[0])
        dl = A.DeviceLayout.from_layout(A.LayeredLayout(
            d["total_layers"], d["layer_offsets"], d["node_ids"], d["row_ptr"], d["in_nodes"],
            d["in_weights"], d["input_order"], 0, d["id_bound"], shard[0].outputs), device=local)
    else:
        dl = A.DeviceLayout.from_network(shard[0], device=local)
    dev.synchronize()
    t_pre = time.perf_counter() - t0
    pre_t = dev.timings()
    info = dl.info()
    plan = dl.plan(B)

    x_dev = torch.from_numpy(np.concatenate([x.reshape(-1) for x in Xs])).cuda()
    my_off = sum(out_counts[:rank])
    out_all = torch.zeros(max(1, sum(out_counts)), dtype=torch.float32, device="cuda")
    out_dev = out_all[my_off:my_off + max(1, out_counts[rank])]
    torch.cuda.synchronize()

    def gather_out():
        if dist is None:
            return
        if one_gpu:
            parts = [torch.zeros(c) for c in out_counts]
            dist.all_gather(parts, out_dev[:out_counts[rank]].cpu())
            out_all.copy_(torch.cat(parts), non_blocking=True)
        elif engine_gather:
            dev.allgather(out_dev.data_ptr(), out_all.data_ptr(), out_counts)
        else:
            mx = max(out_counts)
            pad = torch.zeros(mx, device=out_dev.device)
            pad[:out_counts[rank]] = out_dev[:out_counts[rank]]
            parts = [torch.empty(mx, device=out_dev.device) for _ in out_counts]
            dist.all_gather(parts, pad)
            out_all.copy_(torch.cat([p[:c] for p, c in zip(parts, out_counts)]))

    def step():
        dl.activate_device(x_dev.data_ptr(), B, out_dev.data_ptr())
        gather_out()

    tw = time.perf_counter()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    per_step_s = (time.perf_counter() - tw) / max(1, args.warmup)
    # nvidia-smi samples every 100 ms and needs ~0.1 s to start: a timed
    # region shorter than that is bracketed by 0.3 s of the same (untimed)
    # steps on each side inside the sampler, so the clocks reported are the
    # ones under this load
    pad = 0.0 if per_step_s * args.steps > 0.5 else 0.3

    def load(seconds):
        t_end = time.perf_counter() + seconds
        while time.perf_counter() < t_end:
            for _ in range(16):
                step()
            torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        load(pad)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        load(pad)
    ms = ev0.elapsed_time(ev1) / args.steps

    # per-launch device times (events between launches, same stream), for the
    # dominant kernel's roofline: median over 3 profiled sweeps
    prof = np.median(np.stack([dl.profile(x_dev.data_ptr(), B, out_dev.data_ptr())
                               for _ in range(3)]), axis=0)
    if os.environ.get("ASNN_BENCH_DIAG") and rank == 0:
        pathlib.Path(os.environ["ASNN_BENCH_DIAG"]).write_text(json.dumps(
            {"launch_ms": [float(v) for v in prof], "info": info, "ms_per_step": ms}))

    # check the gathered outputs once (rank 0 holds everything after the gather)
    step()
    torch.cuda.synchronize()
    if dist is not None:
        assert torch.equal(out_all[my_off:my_off + out_counts[rank]], out_dev[:out_counts[rank]])

    # e2e: host (pinned) buffers.  One GPU: the C-ABI call with host pointers
    # (H2D of the batch and D2H of the outputs inside the call).  N GPUs: each
    # rank's H2D of its slice, the sweep, the in-engine gather, and rank 0's
    # D2H of the gathered outputs.
    x_pin = torch.from_numpy(np.concatenate([x.reshape(-1) for x in Xs])).pin_memory()
    out_pin = torch.empty(max(1, sum(out_counts)), dtype=torch.float32).pin_memory()

    # batch <= 64 of one network that fits one SM's shared memory: the
    # resident server (asnn_dev_server_*, csrc/serve.cuh) -- the per-request
    # path without a launch or stream synchronisation
    server = None
    if dist is None and B <= 64 and len(shard) == 1 and not os.environ.get("ASNN_BENCH_NO_SERVER"):
        try:
            server = dl.serve(max_vec=B)
        except (A.BackendUnavailable, ValueError):
            server = None
    e2e_path = ("resident server (asnn_dev_server_activate)" if server is not None else
                "asnn_dev_activate with page-locked host buffers" if dist is None else
                "H2D + sweep + in-engine gather + D2H per rank")

    def e2e_step():
        if server is not None:
            server.activate_ptr(x_pin.data_ptr(), B, x_pin.numel(), out_pin.data_ptr())
        elif dist is None:
            dl.activate_host_ptr(x_pin.data_ptr(), B, x_pin.numel(), out_pin.data_ptr())
        else:
            x_dev.copy_(x_pin, non_blocking=True)
            step()
            if rank == 0:
                out_pin.copy_(out_all, non_blocking=True)
            stream.synchronize()

    e2e_step()
    # (not torch.cuda.synchronize(): a device-wide wait would wait for the
    # resident server, a persistent kernel, to exit)
    stream.synchronize()
    if dist:
        dist.barrier()
    for _ in range(args.warmup):
        e2e_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if server is not None:
        server.close()
    # one vector of one network (C1): also the literal per-call drop-in --
    # the layout staged again and evaluated by one kernel every call
    # (asnn_eval_buf, csrc/once.cu), id-indexed state back
    per_call = None
    if dist is None and B == 1 and len(shard) == 1:
        lay = dl.download(0)
        buf = A.EvalBuffer()
        x1 = Xs[0][0]
        for _ in range(max(3, args.warmup)):
            buf.stage_layout(lay, x1)
            buf.run()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            buf.stage_layout(lay, x1)
            st_out = buf.run()
        pc_s = (time.perf_counter() - t0) / args.steps
        per_call = {"value": sum(len(n.source) for n in nets) / pc_s, "unit": "conn_evals/s",
                    "us_per_step": pc_s * 1e6, "variant": buf.mode,
                    "path": "eval_parallel drop-in: layout staged + one kernel every call "
                            "(asnn_eval_buf, Python API), id-indexed state back",
                    "h2d_bytes_per_step": int(8 * len(lay.in_nodes) + 12 * len(lay.node_ids)),
                    "d2h_bytes_per_step": int(4 * len(st_out))}
        buf.free()

    evaluated = info["edge_count"]
    if dist:
        t = torch.tensor([ms, e2e_s, float(evaluated if cfg == "c5" else 0)], dtype=torch.float64)
        if not one_gpu:
            t = t.cuda()
        red = t.clone()
        dist.all_reduce(red, op=dist.ReduceOp.MAX)
        ms, e2e_s = float(red[0]), float(red[1])
        if cfg == "c5":
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            evaluated = int(t[2])

    E = sum(len(n.source) for n in nets)
    conn_evals_total = E * B_total
    value = conn_evals_total / (ms / 1e3)
    peak, peak_src = measured_peak()
    # level kernels: every launch but the sensor and output-gather ones
    level_ms = float(prof[1:-1].sum()) if len(prof) > 2 else float(prof.sum())
    achieved = plan["alg_bytes"] / (level_ms / 1e3) / 1e9
    # the committed ncu figure is for the full-size, one-GPU sweep only
    traffic = profiled_traffic(cfg) if args.scale == 1.0 and world == 1 and not args.shard_of else None
    cb = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(nets, X, cfg, budget_s=args.cpu_budget)
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "conn_evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if cfg != "c5" else "weak", "vs_baseline": None, "dtype": "f32",
            "data": DATA,
            "config": config_dict(cfg, nets, world),
            # the reference's convention counts every connection (bench.cpp:53);
            # edges into nodes without a level are never evaluated by either side
            "evaluated_edges": int(evaluated),
            "value_evaluated": evaluated * B_total / (ms / 1e3),
            "levels": info["total_layers"],
            "gather": gather,
            "e2e": {"value": conn_evals_total / e2e_s, "unit": "conn_evals/s",
                    "h2d_bytes_per_step": int(sum(x.size for x in X) * 4),
                    "d2h_bytes_per_step": int(sum(out_counts) * 4),
                    "us_per_step": e2e_s * 1e6, "path": e2e_path},
            **({"e2e_per_call": per_call} if per_call else {}),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": peak_src,
                         # what actually binds, when it is not HBM
                         "binding": BINDING.get(cfg),
                         "alg_bytes_per_step": plan["alg_bytes"],
                         # measured DRAM bytes (ncu) over the same launch time: the
                         # bandwidth the HBM actually delivered
                         "dram_frac": (traffic / (level_ms / 1e3) / 1e9 / peak) if traffic else None,
                         # every byte read or written once (edges,
                         # row pointers, each activation written and read once)
                         "compulsory_bytes_per_step": int(8 * E + 4 * (info["node_count"] + 1) +
                                                          8 * info["node_count"] * B),
                         "kernel": {"rows": "k_rows + k_heavy (one launch each per dependency level)",
                                    "segments": "k_rows (heavy rows split across levels) per dependency level",
                                    "k_cta": "k_cta (one CTA per network x batch slice, whole sweep)",
                                    "k_chain": "k_chain (one CTA per batch column, decoupled finish / prefix "
                                               "warps, whole sweep)"}
                                   [plan["strategy"]],
                         "kernel_ms_per_step": level_ms, "launches_per_step": len(prof),
                         "max_launch_ms": float(prof.max()),
                         "sweep_achieved_gbs": plan["alg_bytes"] / (ms / 1e3) / 1e9},
            "cpu_baseline": cb,
            "gpu_launches": plan["kernels"] * args.steps,  # ours only (the gather is NCCL's)
            "clocks": dict(clk.summary(), window="timed region" if not pad else
                           f"timed region + {pad} s of untimed steps on each side"),
            "preprocess": {"wall_s": t_pre, "device_ms": pre_t, "generate_s": t_gen},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


BINDING = {"c4": "HBM random-row gathers (0.92 of the 256-B gather ceiling)",
           "c2": "L2 throughput: gathers served from L2 (DRAM 0.46 GB of 20.8 GB algorithmic), "
                 "so frac > 1 against HBM",
           "c3": "latency: one dependent chain per layer per CTA, 2000 layers",
           "c5": "FP64 sigmoid latency / layer barriers, shared-memory resident",
           "c1": "latency: 10 layers in one CTA"}


def run_reference(args, cfg):
    """The reference arm: the reference's own CPU implementation (oracle/_ref)
    on this box's host cores, on the same workload and config as ours.  Only
    oracle/ is loaded (never the engine).  Each step evaluates a bounded
    sample of the batch's vectors in the fastest of the reference's modes
    (picked on a short calibration); value = connection evals of the timed
    steps / their measured time."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    nets = make_network_ref(cfg, args.scale)
    rng = np.random.default_rng(12345)
    B_total = CONFIGS[cfg][1]
    n_in = [net_counts(n)[1] for n in nets]
    if cfg == "c5":
        X = [rng.uniform(-2, 2, (B_total, k)).astype(np.float32) for k in n_in]
    else:
        X = [rng.uniform(-2, 2, (B_total, n_in[0])).astype(np.float32)]
    cpu = RefCPU(nets, X, cfg)
    calib = cpu.measure(budget_s=max(1.5, args.cpu_budget / 4))
    mode = calib["mode"]
    # vectors per step: about 0.5 s of work per step (whole multiples of the
    # thread count for omp-seq), at most the batch
    per_vec = calib["modes"][mode]["seconds"] / calib["modes"][mode]["vectors"] \
        if "modes" in calib else 1.0
    n_vec = max(1, min(B_total, int(0.5 / max(per_vec, 1e-9))))
    if mode == "omp-seq":
        n_vec = min(B_total, max(cpu.threads, n_vec // cpu.threads * cpu.threads))
    # a sample shorter than ~20 ms (C1: one 10k-connection vector) is timed as
    # the mean of `reps` back-to-back runs of it inside the step
    _, t_sample = cpu.run(mode, n_vec)
    reps = max(1, int(0.02 / max(t_sample, 1e-9))) if t_sample < 0.02 else 1
    times, evs = [], []
    for i in range(args.warmup + args.steps):
        ev = dt = 0.0
        for _ in range(reps):
            e, t = cpu.run(mode, n_vec)
            ev, dt = ev + e, dt + t
        if i >= args.warmup:
            times.append(dt / reps)
            evs.append(ev / reps)
    value = sum(evs) / sum(times)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value, "unit": "conn_evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "ms_per_step": statistics.mean(times) * 1e3, "dtype": "f32",
        "data": DATA,
        "config": config_dict(cfg, nets, world),
        "conn_evals_per_step": int(evs[0]),
        "evaluated_edges": int(cpu.evaluated) if cfg != "c5" else None,
        "cpu_baseline": {"value": value, "unit": "conn_evals/s", "kind": cpu.kind,
                         "cores": 1 if mode == "seq" else cpu.threads, "mode": mode,
                         "modes": calib.get("modes"),
                         "sample": f"each step: {n_vec} of the {B_total} vectors x {cpu.n_nets} "
                                   f"network(s) ({mode}"
                                   + (f", mean of {reps} back-to-back runs" if reps > 1 else "")
                                   + "); mode picked on a calibration run"},
        "e2e": {"value": value, "unit": "conn_evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "vs_baseline": None,
    }
    print(json.dumps(line), flush=True)


def run_ncu_sweeps(args, cfg):
    """Layout build + N plain sweeps (no graph, no timing): the command the
    committed ncu launch lists and captures in profiles/ were taken with."""
    import torch
    import paper_2005_04347_b200 as A
    nets = make_network(cfg, args.scale)
    B = CONFIGS[cfg][1] // max(1, args.shard_of) if cfg != "c5" else CONFIGS[cfg][1]
    rng = np.random.default_rng(12345)
    X = np.concatenate([rng.uniform(-2, 2, (B, len(n.inputs))).astype(np.float32).reshape(-1)
                        for n in nets])
    dl = (A.DeviceLayout.from_population(nets) if cfg == "c5"
          else A.DeviceLayout.from_network(nets[0]))
    x_dev = torch.from_numpy(X).cuda()
    out_dev = torch.empty(dl.info()["n_outputs"] * B, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    for _ in range(args.ncu_sweeps):
        dl.profile(x_dev.data_ptr(), B, out_dev.data_ptr())
    torch.cuda.synchronize()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scale", type=float, default=1.0, help="shrink c4/c5 for quick runs")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--shard-of", type=int, default=0,
                    help="development: run rank 0's batch slice of a G-GPU split on this one GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--prep", default="device", choices=["device", "upload"],
                    help="device: compute_required/segment/flatten on the GPU; upload: "
                         "asnn_dev_upload_layout of the generator's banded layout")
    ap.add_argument("--ncu-sweeps", type=int, default=0,
                    help="profiling helper: build the layout, run this many sweeps, print "
                         "nothing else (for ncu launch lists; never a bench number)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not args.ncu_sweeps:
        # one process per GPU: re-launch this command under torchrun
        import socket
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", str(pathlib.Path(__file__).resolve())] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.ncu_sweeps:
        run_ncu_sweeps(args, args.config)
    elif args.impl == "reference":
        run_reference(args, args.config)
    else:
        run_ours(args, args.config)


if __name__ == "__main__":
    main()

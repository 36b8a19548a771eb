"""Benchmark driver (contract: the round's README / SURVEY.md section 8(d)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tnb|reference]
                    [--no-secondary] [--no-cpu]

Headline workload (BASELINE.json configs[2], f64 part, the north-star target):
L.A.W.R effective-Hamiltonian matvec through ``Network.launch`` at chi=1024, d=2,
D=5, float64, optimal order (((A,L),W),R); metric fp64 GFLOP/s (algorithmic
2*MACs from the reference's own cost model). The other BASELINE configs are
measured in the same run and reported, compactly, under "workloads" (full
detail in gpurun_out/bench_detail.json when that directory exists). Inputs are
the reference recipes' seeded N(0,1)/U(0,1) synthetic tensors -- there is no
dataset. Every workload's output is checked (untimed) against the CPU oracle
(oracle/tnkit_np.py, the checker only) and the error is printed as "par".

--gpus N without torchrun re-launches this script under torch.distributed.run
with N ranks (one process per GPU, NCCL). The single matvec and the permute
sweep are replicated per rank (weak scaling); the C3b batch, the C4 batch and
the C5 sites are sharded by unit over the ranks (strong scaling of the batch);
one C4 contraction is also partitioned by output panels + one NCCL all-gather.

--impl reference times the reference algorithm's CPU path (the numpy port in
oracle/, the same numpy/OpenBLAS calls as the reference's tnkit) on this
host's cores, rank 0 only.
"""
import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np

FP64_PEAK_TFLOPS = 37.06   # measured DMMA peak on this pool's B200 (profiles/r01_fp64_peak.txt)
PEAK_SOURCE = "DMMA.8x8x4 microbenchmark, profiles/r01_fp64_peak.txt (no fp64 in MEASURED_PEAKS.json)"
METRIC = "fp64 GFLOP/s (L.A.W.R Network matvec, chi=1024)"
CONFIG = {"workload": "lawr_f64_chi1024", "chi": 1024, "d": 2, "D": 5, "order": "(((A,L),W),R)"}
DATA = "synthetic (seeded N(0,1), reference recipe)"
TOL = 1e-12


def peaks():
    hbm = 6546.9
    src = "fallback"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        hbm = float(mp.get("hbm_gbs", hbm))
        src = "MEASURED_PEAKS.json"
    except Exception:
        pass
    return hbm, src


def traffic_per_launch(kernel, dtype):
    """DRAM bytes (read + write) per launch of `kernel` from the committed `ncu --set full`
    capture of this workload (profiles/*_traffic.json, newest round first), or None."""
    for name in ("r02_traffic.json", "r01_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                tr = json.load(f)
        except Exception:
            continue
        key = f"{kernel}:{np.dtype(dtype).name}"
        if key in tr:
            return tr[key]["bytes_per_launch"]
    return None


def host_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = None
    return {"cpu": model, "cpu_count": os.cpu_count(), "affinity": aff, "blas_threads": cpu_threads()}


# ----------------------------------------------------------------------------- dist
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = "nccl"

    def init(self, backend):
        # dev: TNB_BENCH_BACKEND=gloo runs the multi-rank code paths with host-side
        # collectives (e.g. two ranks sharing one GPU) -- a functional check, not a measurement
        self.backend = os.environ.get("TNB_BENCH_BACKEND", backend)
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=self.backend)
            self.pg = dist

    @property
    def coll_device(self):
        import torch
        return "cuda" if torch.cuda.is_available() and self.backend == "nccl" else "cpu"

    def barrier(self):
        if self.pg:
            if self.coll_device == "cuda":
                self.pg.barrier(device_ids=[self.local])
            else:
                self.pg.barrier()

    def all_gather(self, out, inp):
        """all_gather_into_tensor, staged through host memory for a host backend."""
        if self.coll_device == "cuda" or not inp.is_cuda:
            self.pg.all_gather_into_tensor(out, inp)
            return
        o = out.cpu()
        self.pg.all_gather_into_tensor(o, inp.cpu())
        out.copy_(o)

    def _reduce(self, x, op):
        if not self.pg:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64, device=self.coll_device)
        self.pg.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x):
        return self._reduce(x, self.pg.ReduceOp.MAX) if self.pg else x

    def sum(self, x):
        return self._reduce(x, self.pg.ReduceOp.SUM) if self.pg else x


def relaunch(args):
    """`--gpus N` outside torchrun: run this script under torch.distributed.run with N ranks
    (one process per GPU) on 127.0.0.1; rank 0's JSON line passes through."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")            # comm init lines (nranks) for the record ...
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr, never in the JSON stdout
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- timing
def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


class L2Flush:
    """Write a 256 MiB buffer (> 126 MB L2), then read another one: the reads evict the
    dirty lines of the write, so the timed kernel starts with a cold AND clean L2."""
    def __init__(self):
        import torch
        self.buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        self.rd = torch.ones(32 << 20, dtype=torch.float64, device="cuda")

    def __call__(self):
        self.buf.zero_()
        self.rd.sum()


class _NoGC:
    """Python's cyclic GC collected before and paused inside a timed region (as timeit):
    a generation-2 pass over a large heap is a 10-40 ms host stall unrelated to the work."""
    def __enter__(self):
        import gc
        gc.collect()
        self.was = gc.isenabled()
        gc.disable()

    def __exit__(self, *a):
        import gc
        if self.was:
            gc.enable()


WARM_UNTIMED = 2  # untimed steps time_steps runs first (the kernel timer sees them too)


def time_steps(fn, steps, flush, dist, warm=WARM_UNTIMED):
    """Device time of `steps` calls of fn, each bracketed by its own events; L2 flushed
    (untimed) before every call; barrier + synchronize around the region; max over ranks."""
    import torch
    pairs = []
    dist.barrier()
    torch.cuda.synchronize()
    with _NoGC():
        # two untimed steps first: the GPU would otherwise enter the first timed step from the
        # idle gap of the barrier / synchronize above (measured: +0.14 ms on the headline's
        # first step, +0.9-1.6 ms on C3 c128's, every later step level)
        for _ in range(warm):
            flush()
            fn()
        for _ in range(steps):
            flush()
            e0, e1 = _events()
            e0.record()
            fn()
            e1.record()
            pairs.append((e0, e1))
        torch.cuda.synchronize()
    dist.barrier()
    each = [a.elapsed_time(b) for a, b in pairs]
    _LAST_STEPS[:] = each
    return dist.max(sum(each))


_LAST_STEPS = []  # per-step ms of the last time_steps call (detail only)


def time_region(fn, dist):
    """Device time of ONE call of fn (a whole loop), events around it, max over ranks."""
    import torch
    dist.barrier()
    torch.cuda.synchronize()
    with _NoGC():
        e0, e1 = _events()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
    dist.barrier()
    return dist.max(e0.elapsed_time(e1))


def ktimer(tnb, fn, *families):
    """Run fn with the library's kernel timer on (CUDA event pair around each libtnb launch
    on the stream it is launched on); returns [(launches, ms, work)] per family."""
    tnb._lib.ktimer_reset()
    tnb._lib.ktimer_enable(True)
    try:
        fn()
    finally:
        tnb._lib.ktimer_enable(False)
    out = [tnb._lib.ktimer_read(f) for f in families]
    tnb._lib.ktimer_reset()
    return out


def roofline_tensor(achieved_tflops, kernel, traffic=None):
    return {"bound": "tensor", "achieved": round(achieved_tflops, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": round(achieved_tflops / FP64_PEAK_TFLOPS, 4), "traffic": traffic, "kernel": kernel}


def rel_err(got, want):
    got, want = np.asarray(got), np.asarray(want)
    den = float(np.linalg.norm(want.reshape(-1)))
    num = float(np.linalg.norm((got - want).reshape(-1)))
    return num / den if den > 0 else num


# ----------------------------------------------------------------------------- GPU workloads
def make_network(tnb, lines, arrays):
    net = tnb.Network(lines)
    tensors = {}
    for nm, arr in arrays.items():
        t = tnb.UniTensor(tnb.storage.from_numpy(arr), labels=[f"x{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
        tensors[nm] = t
    net.set_order(optimal=True)
    return net, tensors


def lawr_macs(tnb, chi, d=2, D=5):
    sets, dims = WL.lawr_label_sets(), WL.lawr_dims(chi, d, D)
    tree = tnb.find_optimal_order(sets, dims)
    return tnb.contraction_cost(tree, sets, dims), tnb.render_order(tree)


E2E_CHUNKS = int(os.environ.get("TNB_E2E_CHUNKS", "2"))  # 1-8 swept with double buffering: 2 best
E2E_SETS = int(os.environ.get("TNB_E2E_SETS", "3"))      # buffer sets rotated by the serving loop (3: 1.907 vs 1.931 ms)


def lawr_e2e(tnb, inp, order, steps, warmup, dist, flop, graph=False):
    """End to end through the public API: pinned host inputs -> HBM (upload_), launch, result
    streamed back to pinned host memory (launch(host_out=...)) every step. A serving loop:
    two networks with their own device inputs and pinned host buffers alternate, each refill
    ordered only after the launch that last read that set, so step i+1's uploads overlap step
    i's kernels."""
    import torch
    sets = [make_network(tnb, WL.LAWR_NET, inp) for _ in range(E2E_SETS)]
    pinned = [{nm: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for nm, a in inp.items()} for _ in sets]
    h2d = sum(p.numel() * p.element_size() for p in pinned[0].values())
    probe = sets[0][0].launch().get_block_().contiguous().storage()
    outs = [torch.empty(probe.shape, dtype=probe.dtype, pin_memory=True) for _ in sets]
    first_use = tnb.tree_leaves(tnb.parse_order(order))

    def step(i):
        n, ts = sets[i % E2E_SETS]
        for nm in first_use:
            big = pinned[0][nm].numel() * pinned[0][nm].element_size() >= (8 << 20)
            ts[nm].get_block_().upload_(pinned[i % E2E_SETS][nm], chunks=E2E_CHUNKS if big else 1,
                                        after=n.done_event)
        n.launch(host_out=outs[i % E2E_SETS])

    def loop(k):
        return lambda: [step(i) for i in range(k)]
    if graph:
        # latency-bound sizes: each buffer set's whole step (input uploads, the launch, the
        # result copy to its pinned buffer) captured once as a CUDA graph and replayed on the
        # set's own stream -- one graph launch per step instead of the per-call host work
        cur = torch.cuda.current_stream()
        streams = [torch.cuda.Stream() for _ in sets]
        graphs = []
        for k, (n, ts) in enumerate(sets):
            def step_k(n=n, ts=ts, k=k):
                for nm in first_use:
                    big = pinned[0][nm].numel() * pinned[0][nm].element_size() >= (8 << 20)
                    ts[nm].get_block_().upload_(pinned[k][nm], chunks=E2E_CHUNKS if big else 1)
                return n.launch(host_out=outs[k])
            with torch.cuda.stream(streams[k]):
                graphs.append(tnb.graphs.capture(step_k))
        torch.cuda.synchronize()

        def gstep(i):
            k = i % E2E_SETS
            streams[k].wait_stream(cur)
            with torch.cuda.stream(streams[k]):
                graphs[k].replay()

        def loop(k):  # noqa: F811
            def run():
                for i in range(k):
                    gstep(i)
                for st_ in streams:
                    cur.wait_stream(st_)
            return run
    time_region(loop(max(2, warmup)), dist)
    ems = time_region(loop(steps), dist)
    lat = time_region(loop(1), dist)
    d2h = outs[0].numel() * outs[0].element_size()
    e2e = {"value": round(dist.sum(flop) / (ems / steps) / 1e6, 3), "unit": "GFLOP/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ems / steps, 4),
           "single_step_latency_ms": round(lat, 4)}
    if graph:
        e2e["api"] = "graphs.capture(upload_ per input, Network.launch(host_out=...)) per buffer set"
    # every set's host result is the network's output (a chunk-uploaded operand computes the
    # root step panel by panel: other stream-K splits, so equal to rounding, not bit for bit)
    torch.cuda.synchronize()
    want = probe.cpu().numpy()
    e2e["host_result_rel_err"] = _r(max(rel_err(o.reshape(want.shape).numpy(), want) for o in outs), 3)
    return e2e


def gpu_lawr(tnb, chi, dtype, steps, warmup, flush, dist, e2e=True, graph=False, seed=1234, e2e_graph=False):
    """One L.A.W.R matvec per step (replicated per rank, weak scaling)."""
    import torch
    inp = WL.lawr_inputs(chi, dtype=dtype, seed=seed)  # same instance on every rank (replicas)
    net, _ = make_network(tnb, WL.LAWR_NET, inp)
    macs, order = lawr_macs(tnb, chi)
    flop = macs * (8 if dtype == np.complex128 else 2)
    for _ in range(warmup):
        net.launch()
    l0 = tnb._lib.launch_count()
    m0 = torch.cuda.memory_stats()
    ms = time_steps(net.launch, steps, flush, dist)
    m1 = torch.cuda.memory_stats()
    each = [round(x, 4) for x in _LAST_STEPS]
    allocs = {k: m1.get(k, 0) - m0.get(k, 0) for k in ("num_device_alloc", "num_device_free", "num_alloc_retries")}
    launches = (tnb._lib.launch_count() - l0) // max(steps, 1)
    assert net.get_order() == order
    out = net.launch().numpy()
    res = {"ms_per_step": ms / steps, "ms_each_step": each, "allocator": allocs, "flop_per_step": flop, "order": order,
           "launches_per_step": launches,
           "gflops": dist.sum(flop) / (ms / steps) / 1e6, "out": out, "inp": inp}
    if graph:
        cn = net.compile()
        for _ in range(warmup):
            cn.launch()
        gms = time_steps(cn.launch, steps, flush, dist) / steps
        res["graph_ms_per_step"] = gms
        res["gflops_graph"] = dist.sum(flop) / gms / 1e6
    if e2e:
        if e2e_graph or os.environ.get("TNB_E2E_GRAPH"):
            res["e2e"] = lawr_e2e(tnb, inp, order, steps, warmup, dist, flop, graph=True)
            res["e2e_eager"] = lawr_e2e(tnb, inp, order, steps, warmup, dist, flop)
        else:
            res["e2e"] = lawr_e2e(tnb, inp, order, steps, warmup, dist, flop)
    # dominant kernel = the stream-K DMMA GEMM (A.L and T2.R): kernel timer over the same
    # timed region (flush, K steps)
    (n_g, ms_g, fl_g), (n_s, ms_s, _) = ktimer(tnb, lambda: time_steps(net.launch, steps, flush, dist),
                                               tnb._lib.KF_GEMM, tnb._lib.KF_GEMM_SKINNY)
    ach = fl_g / (dist.max(ms_g) / 1e3) / 1e12 if n_g else 0.0
    ks = steps + WARM_UNTIMED  # steps the kernel timer saw
    res["steps_ms"] = {"gemm": round(ms_g / ks, 4), "skinny_T1W": round(ms_s / ks, 4),
                       "gemm_launches_per_step": n_g / ks, "gemm_share_of_step": round((ms_g / ks) / (ms / steps), 4)}
    res["roofline"] = roofline_tensor(ach, "gemm_sk_kernel (stream-K DMMA.8x8x4), steps A.L + T2.R",
                                      traffic_per_launch("gemm_sk_kernel", dtype))
    res["roofline_how"] = ("achieved = algorithmic flop of the GEMM launches / their summed CUDA-event durations on "
                           "the launching stream, over the K timed steps; peak: " + PEAK_SOURCE)
    return res


def gpu_lawr_batch(tnb, n_total, chi, dtype, steps, warmup, flush, dist):
    """C3b: a batch of independent L.A.W.R matvecs (seeds 5000 + 4i), sharded by instance."""
    import torch
    from paper_2401_01921_b200 import parallel
    mine = parallel.shard(n_total, dist.world, dist.rank)
    nets, inps = [], []
    for i in mine:
        inp = WL.lawr_inputs(chi, dtype=dtype, seed=WL.lawr_batch_seed(i))
        nets.append(make_network(tnb, WL.LAWR_NET, inp))
        inps.append(inp)
    macs, order = lawr_macs(tnb, chi)
    flop = macs * (8 if dtype == np.complex128 else 2)

    def step():
        for net, _ in nets:
            net.launch()
    for _ in range(warmup):
        step()
    ms = time_steps(step, steps, flush, dist) / steps
    ((n_g, ms_g, fl_g),) = ktimer(tnb, lambda: time_steps(step, steps, flush, dist), tnb._lib.KF_GEMM)
    ach = fl_g / (dist.max(ms_g) / 1e3) / 1e12 if n_g else 0.0
    res = {"ms_per_step": ms, "instances": n_total, "per_rank": len(mine), "gflops": flop * n_total / ms / 1e6,
           "roofline": roofline_tensor(ach, "gemm_sk_kernel, complex128 4M")}
    # e2e: every instance's inputs from pinned host memory, result back to pinned host memory
    pinned = [{nm: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for nm, a in inp.items()} for inp in inps]
    probe = nets[0][0].launch().get_block_().contiguous().storage()
    outs = [torch.empty(probe.shape, dtype=probe.dtype, pin_memory=True) for _ in nets]
    first_use = tnb.tree_leaves(tnb.parse_order(order))

    def e2e_step():
        for (net, ts), pin, out in zip(nets, pinned, outs):
            for nm in first_use:
                ts[nm].get_block_().upload_(pin[nm], after=net.done_event)
            net.launch(host_out=out)
    e2e_step()
    ems = time_region(e2e_step, dist)
    h2d = sum(p.numel() * p.element_size() for pin in pinned for p in pin.values())
    d2h = sum(o.numel() * o.element_size() for o in outs)
    res["e2e"] = {"value": round(flop * n_total / ems / 1e6, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
                  "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ems, 3)}
    torch.cuda.synchronize()
    res["out0"] = outs[0].numpy().reshape(chi, 2, chi) if 0 in mine else None
    return res


def gpu_permute(tnb, steps, warmup, flush, dist, check=True):
    """C2: every permutation of the sweep, t.permute(*p).contiguous(). Value = bytes moved by
    K permutes replayed BACK TO BACK from a CUDA graph after one L2 flush (each permute pays
    the previous one's dirty-line write-back: steady state), median over permutations."""
    import itertools
    out, samples = {}, []
    for shape, dt, name in [((64,) * 4, np.float64, "r4_f64"), ((64,) * 4, np.complex128, "r4_c128"),
                            ((16,) * 6, np.float64, "r6_f64"), ((16,) * 6, np.complex128, "r6_c128")]:
        src = tnb.storage.uniform(list(shape), dtype=dt, seed=11)
        if len(shape) == 4:
            perms = [p for p in itertools.permutations(range(4)) if p != (0, 1, 2, 3)]
        else:
            g = np.random.default_rng(606)
            perms = []
            while len(perms) < 32:
                p = tuple(int(x) for x in g.permutation(6))
                if p != tuple(range(6)):
                    perms.append(p)
        nbytes = 2 * src.size * src.itemsize
        k = max(4, steps)
        rates, single = [], []
        for p in perms:
            g = tnb.graphs.capture(lambda: src.permute(*p).contiguous(), warmup=max(1, warmup // 2))
            ms = time_steps(lambda: [g.replay() for _ in range(k)], 1, flush, dist)
            rates.append(nbytes * k / ms / 1e6)
            ms1 = time_steps(g.replay, 2, flush, dist) / 2  # one permute from a flushed L2
            single.append(nbytes / ms1 / 1e6)
            if check and p == perms[len(perms) // 2]:
                samples.append((name, shape, dt, p, g.output.numpy()))
            del g
        out[name] = {"median_gbs": float(np.median(rates)), "min_gbs": float(np.min(rates)),
                     "max_gbs": float(np.max(rates)), "single_flushed_median_gbs": float(np.median(single)),
                     "n_perms": len(perms), "bytes_per_permute": nbytes}
    return out, samples


def c4_tensors(tnb, seed=777):
    u1 = tnb.Symmetry.u1()
    V = tnb.Bond(btype=tnb.IN, sectors=WL.c4_sectors(), syms=[u1])
    P = tnb.Bond(btype=tnb.IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    A = tnb.UniTensor([V, P, V.redirect()], labels=["vl", "p", "vr"])
    E = tnb.UniTensor([V, P.redirect(), V.redirect()], labels=["vr", "p", "x"])
    tnb.random.normal_(A, seed=seed)
    tnb.random.normal_(E, seed=seed + 1)
    return A, E


C4_MACS = 169073208


def gpu_c4(tnb, steps, warmup, flush, dist):
    """C4: one U(1) block-sparse contract(A, E) per step (replicated per rank); plus, at N>1,
    the same contraction partitioned over the ranks (strong scaling of one call)."""
    import torch
    A, E = c4_tensors(tnb)
    for _ in range(warmup):
        tnb.contract(A, E)
    ms = time_steps(lambda: tnb.contract(A, E), steps, flush, dist) / steps
    g = tnb.graphs.capture(lambda: tnb.contract(A, E))
    gms = time_steps(g.replay, steps, flush, dist) / steps
    ((n_k, ms_k, _),) = ktimer(tnb, lambda: time_steps(lambda: tnb.contract(A, E), steps, flush, dist),
                               tnb._lib.KF_BS_GEMM)
    kms = dist.max(ms_k / max(n_k, 1))
    res = {"ms_per_call_eager": ms, "ms_per_call_graph": gms, "bs_gemm_kernel_ms": kms,
           "gflops_eager": dist.sum(2 * C4_MACS) / ms / 1e6, "gflops": dist.sum(2 * C4_MACS) / gms / 1e6,
           "roofline": roofline_tensor(2 * C4_MACS / kms / 1e9, "bs_sk_kernel (grouped stream-K DMMA.8x8x4)",
                                       traffic_per_launch("bs_sk_kernel", np.float64))}
    # e2e: A and E payloads (packed .utn layout) from pinned host memory, result payload back
    from paper_2401_01921_b200 import io as tio
    hA = torch.empty(tio.payload_nbytes(A), dtype=torch.uint8, pin_memory=True)
    hE = torch.empty(tio.payload_nbytes(E), dtype=torch.uint8, pin_memory=True)
    tio.download_payload(A, hA)
    tio.download_payload(E, hE)
    out = tnb.contract(A, E)
    # a serving loop over E2E_SETS device tensor sets of the same structure. Each set's whole
    # step -- both payload uploads (pinned host -> staging -> scatter into the slabs), the
    # contraction, the result payload download -- is captured once as a CUDA graph
    # (graphs.capture over the public payload / contract calls) and replayed on the set's own
    # stream, so step i+1's uploads overlap step i's kernel and the host issues one graph
    # launch per step instead of ~10 engine calls (eager serving loop: 0.29-0.35 ms/step,
    # host-bound; kept in the detail as e2e_eager).
    sets = [c4_tensors(tnb, seed=1 + k) for k in range(E2E_SETS)]
    hOs = [torch.empty(tio.payload_nbytes(out), dtype=torch.uint8, pin_memory=True) for _ in sets]
    streams = [torch.cuda.Stream() for _ in sets]
    graphs = []
    for k, (A2, E2) in enumerate(sets):
        def step_k(A2=A2, E2=E2, hO=hOs[k]):
            A2.upload_payload_(hA)
            E2.upload_payload_(hE)
            return tnb.contract(A2, E2).download_payload(hO)
        with torch.cuda.stream(streams[k]):
            graphs.append(tnb.graphs.capture(step_k))
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()

    def e2e_step(i):
        k = i % E2E_SETS
        streams[k].wait_stream(cur)  # (a no-op dependency: the region's start event)
        with torch.cuda.stream(streams[k]):
            graphs[k].replay()

    def loop(n):
        def run():
            for i in range(n):
                e2e_step(i)
            for st_ in streams:
                cur.wait_stream(st_)
        return run
    time_region(loop(max(2, warmup)), dist)
    ems = time_region(loop(steps), dist) / steps
    lat = time_region(loop(1), dist)
    res["e2e"] = {"value": round(dist.sum(2 * C4_MACS) / ems / 1e6, 3), "unit": "GFLOP/s",
                  "h2d_bytes_per_step": int(hA.numel() + hE.numel()), "d2h_bytes_per_step": int(hOs[0].numel()),
                  "ms_per_step": round(ems, 4), "single_step_latency_ms": round(lat, 4),
                  "api": "graphs.capture(upload_payload_ x2, contract, download_payload) per buffer set"}
    # the eager serving loop through the same calls (host-issued every step)
    read = [None] * E2E_SETS
    landed = [torch.cuda.Event() for _ in sets]

    def eager_step(i):
        k = i % E2E_SETS
        A2, E2 = sets[k]
        A2.upload_payload_(hA, after=read[k])
        E2.upload_payload_(hE, after=read[k])
        o = tnb.contract(A2, E2)
        ev = read[k] = torch.cuda.Event()
        ev.record()
        o.download_payload(hOs[k], done=landed[k])

    def eloop(n):
        return lambda: [eager_step(i) for i in range(n)]
    time_region(eloop(max(2, warmup)), dist)
    eems = time_region(eloop(steps), dist) / steps
    res["e2e_eager"] = {"value": round(dist.sum(2 * C4_MACS) / eems / 1e6, 3), "ms_per_step": round(eems, 4)}
    A2, E2 = sets[0]
    torch.cuda.synchronize()
    ref = torch.empty_like(hOs[0])
    tio.download_payload(out, ref)
    torch.cuda.synchronize()
    res["e2e"]["payload_bit_exact"] = all(bool(torch.equal(h, ref)) for h in hOs)
    res["out_blocks"] = [b.numpy() for b in tnb.contract(A2, E2).get_blocks_()]
    if dist.world > 1:
        from paper_2401_01921_b200 import parallel
        for _ in range(warmup):
            parallel.contract_sharded(A, E)
        sms = time_steps(lambda: parallel.contract_sharded(A, E), steps, flush, dist) / steps
        res["sharded"] = {"ms_per_call": sms, "gflops": 2 * C4_MACS / sms / 1e6,
                          "scaling": "strong (one contraction: LPT output panels per rank + NCCL all-gather)"}
        sh = parallel.contract_sharded(A, E)
        res["sharded_par"] = max(rel_err(x.numpy(), y.numpy()) for x, y in
                                 zip(sh.get_blocks_(), tnb.contract(A, E).get_blocks_()))
    return res


def gpu_c4_batch(tnb, n_total, steps, warmup, flush, dist):
    """A batch of independent C4 contractions (e.g. the equal-structure sites of a sweep),
    sharded by unit across ranks (no data-path collective): strong scaling of the batch."""
    from paper_2401_01921_b200 import parallel
    mine = parallel.shard(n_total, dist.world, dist.rank)
    pairs = [c4_tensors(tnb, seed=777 + 2 * i) for i in mine]

    def step():  # ONE grouped launch over the output tiles of all of this rank's contractions
        return tnb.contract_batched(pairs)
    for _ in range(warmup):
        step()
    ms = time_steps(step, steps, flush, dist) / steps
    ((n_k, ms_k, _),) = ktimer(tnb, lambda: time_steps(step, steps, flush, dist), tnb._lib.KF_BS_GEMM)
    kms = dist.max(ms_k / max(n_k, 1))  # (one grouped launch per step)
    res = {"ms_per_step": ms, "instances": n_total, "per_rank": len(mine),
           "gflops": 2 * C4_MACS * n_total / ms / 1e6, "api": "contract_batched (tnb_bs_execute_batched)",
           "bs_gemm_kernel_ms": kms,
           "roofline": roofline_tensor(2 * C4_MACS * len(mine) / kms / 1e9 if kms else 0.0,
                                       "bs_sk_kernel, batched (one launch per rank)")}
    res["out0_blocks"] = [b.numpy() for b in step()[0].get_blocks_()] if 0 in mine else None
    return res


def gpu_peps(tnb, n_sites, chi, D, d, steps, warmup, flush, dist):
    """C5 (reading A): 32 distinct PEPS double-layer site networks (seeds per site), optimal
    order, sharded by site; at N>1 the 32 scalars are all-gathered (NCCL) inside the step."""
    import torch
    from paper_2401_01921_b200 import parallel
    mine = parallel.shard(n_sites, dist.world, dist.rank)
    nets = [make_network(tnb, WL.PEPS_NET, WL.peps_inputs(chi, D, d, site=s))[0] for s in mine]
    shapes = WL.peps_shapes(chi, D, d)
    sets = {n: ls for n, ls in nets[0]._slots}
    dims = {l: dd for nm, ls in nets[0]._slots for l, dd in zip(ls, shapes[nm])}
    tree = tnb.find_optimal_order(sets, dims)
    flop = 2 * tnb.contraction_cost(tree, sets, dims)
    vals = torch.zeros(n_sites, dtype=torch.float64, device="cuda")
    per = (n_sites + dist.world - 1) // dist.world
    mine_buf = torch.zeros(per, dtype=torch.float64, device="cuda")

    def step():
        for k, net in enumerate(nets):
            mine_buf[k:k + 1].copy_(net.launch().get_block_().storage().reshape(-1))
        if dist.pg:
            gathered = torch.empty(per * dist.world, dtype=torch.float64, device="cuda")
            dist.all_gather(gathered, mine_buf)
            # rank r holds sites r, r + world, ...: scatter back to site order
            vals.copy_(gathered.view(dist.world, per).t().reshape(-1)[:n_sites])
        else:
            vals.copy_(mine_buf[:n_sites])
    for _ in range(max(1, warmup)):
        step()
    ms = time_steps(step, steps, flush, dist, warm=0) / steps  # (0.5 s steps: warm-up above suffices)
    ((n_g, ms_g, fl_g),) = ktimer(tnb, lambda: time_steps(step, 1, flush, dist, warm=0), tnb._lib.KF_GEMM)
    ach = fl_g / (dist.max(ms_g) / 1e3) / 1e12 if n_g else 0.0
    return {"ms_per_step": ms, "sites": n_sites, "per_rank": len(mine), "order": tnb.render_order(tree),
            "flop_per_site": flop, "gflops": flop * n_sites / ms / 1e6,
            "roofline": roofline_tensor(ach, "gemm_sk_kernel (all GEMM launches of a site)"),
            "site0": float(vals[0].item()), "gathered": dist.world > 1}


def c4_two_site(tnb, seed=5):
    """(f)3 workload: a two-site U(1) wavefunction on the C4 bonds, psi[vl, p1, p2, vr],
    rowrank 2 -> 23 charge sectors up to 516 x 516 (1.5M stored elements)."""
    u1 = tnb.Symmetry.u1()
    V = tnb.Bond(btype=tnb.IN, sectors=WL.c4_sectors(), syms=[u1])
    P = tnb.Bond(btype=tnb.IN, sectors=[(1, 1), (-1, 1)], syms=[u1])
    psi = tnb.UniTensor([V, P, P, V.redirect()], labels=["vl", "p1", "p2", "vr"], name="psi", rowrank=2)
    tnb.random.normal_(psi, seed=seed)
    return psi


def gpu_svd(tnb, steps, warmup, flush, dist):
    psi = c4_two_site(tnb)
    fn = lambda: tnb.linalg.svd_truncate(psi, keepdim=1024)  # noqa: E731
    for _ in range(max(1, warmup)):
        fn()
    ms = time_steps(fn, steps, flush, dist) / steps
    return {"ms_per_call": ms, "keepdim": 1024, "sectors": 23,
            "note": "one launch of the batched one-sided Jacobi kernel (tnb_svd_jacobi_batched)"}


LANCZOS_ITERS = 30


def gpu_lanczos(tnb, chi, dist):
    """(f)1+(f)2: Lanczos iterations on the Hermitian L.A.W.R effective Hamiltonian at chi,
    matvec = the compiled Network replayed as a CUDA graph. Fixed iteration count so GPU
    and CPU time the same work: ms per Lanczos iteration."""
    import torch
    from paper_2401_01921_b200 import eig
    inp = ORACLE.hermitian_lawr_inputs(chi, seed=7)
    net, _ = make_network(tnb, WL.LAWR_NET, inp)
    op = eig.NetworkMatvec(net.compile(), "A")
    v0 = torch.from_numpy(np.ascontiguousarray(inp["A"]).reshape(-1)).cuda()

    def run():
        try:
            eig.lanczos(op, k=1, v0=v0, tol=1e-14, max_iter=LANCZOS_ITERS, seed=3)
        except eig.ConvergenceError:
            pass
    run()
    ms = time_region(run, dist)
    return {"ms_per_iteration": ms / LANCZOS_ITERS, "iterations": LANCZOS_ITERS, "chi": chi}


def gpu_utn(tnb, steps, warmup, dist):
    """(f)4: .utn load of the C4 MPS tensor A (6.1 MB payload) from the page cache into HBM."""
    import tempfile
    import torch
    A, _ = c4_tensors(tnb)
    path = os.path.join(tempfile.gettempdir(), f"tnb_c4_A_{dist.rank}.utn")
    tnb.save_unitensor(A, path)
    nbytes = sum(b.size * b.itemsize for b in A.get_blocks_())
    for _ in range(max(1, warmup)):
        tnb.load_unitensor(path)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        tnb.load_unitensor(path)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / steps * 1e3
    return {"ms_per_load": ms, "payload_bytes": nbytes, "gbs": nbytes / ms / 1e6, "path": path}


# ----------------------------------------------------------------------------- CPU side
def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads") for i in threadpool_info() if i.get("internal_api") == "openblas"]
        return int(n[0]) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def _best_of(fn, budget_s, max_iter):
    fn()  # warm
    ts = []
    t_start = time.perf_counter()
    while len(ts) < max_iter and (time.perf_counter() - t_start) < budget_s:
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), len(ts)


def cpu_lawr(chi, dtype, budget_s=4.0, max_iter=10, seed=1234):
    inp = ORACLE.lawr_inputs(chi, dtype=dtype, seed=seed)
    sets, dims = WL.lawr_label_sets(), WL.lawr_dims(chi)
    macs = ORACLE.contraction_cost(ORACLE.find_optimal_order(sets, dims), sets, dims)
    flop = macs * (8 if dtype == np.complex128 else 2)
    best, n = _best_of(lambda: ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", inp), budget_s, max_iter)
    return {"value": round(flop / best / 1e9, 3), "unit": "GFLOP/s", "cores": cpu_threads(), "kind": "port",
            "sample": f"{n} Network launches of L.A.W.R chi={chi} {np.dtype(dtype).name} (oracle port of tnkit, "
                      f"numpy {np.__version__} OpenBLAS), best-of", "ms_per_launch": round(best * 1e3, 3)}


def cpu_lawr_batch(n_total, chi, dtype, n_sample=4):
    sets, dims = WL.lawr_label_sets(), WL.lawr_dims(chi)
    macs = ORACLE.contraction_cost(ORACLE.find_optimal_order(sets, dims), sets, dims)
    flop = macs * (8 if dtype == np.complex128 else 2)
    inps = [ORACLE.lawr_inputs(chi, dtype=dtype, seed=WL.lawr_batch_seed(i)) for i in range(n_sample)]
    ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", inps[0])
    t0 = time.perf_counter()
    for inp in inps:
        ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", inp)
    per = (time.perf_counter() - t0) / n_sample
    return {"value": round(flop / per / 1e9, 3), "unit": "GFLOP/s", "cores": cpu_threads(), "kind": "port",
            "sample": f"{n_sample} of the {n_total} instances timed, rate extrapolated linearly to the batch",
            "ms_per_instance": round(per * 1e3, 2)}


def cpu_permute(budget_s=6.0):
    import itertools
    src = ORACLE.uniform([64] * 4, seed=11)
    perms = [p for p in itertools.permutations(range(4)) if p != (0, 1, 2, 3)]
    rates = []
    t_start = time.perf_counter()
    for p in perms:
        if time.perf_counter() - t_start > budget_s:
            break
        t0 = time.perf_counter()
        ORACLE.permute_contiguous(src, p)
        rates.append(2 * src.nbytes / (time.perf_counter() - t0) / 1e9)
    return {"value": round(float(np.median(rates)), 3), "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"{len(rates)} of the 23 rank-4 [64]^4 f64 permutes (np.ascontiguousarray, single-threaded)"}


def c4_oracle_inputs(seed=777):
    sec = ORACLE.c4_sectors()
    qv = [(q,) for q, _ in sec]
    deg = [d for _, d in sec]
    a_qns = ORACLE.zero_flux_combos([(1, qv, [0]), (1, [(1,), (-1,)], [0]), (-1, qv, [0])])
    e_qns = ORACLE.zero_flux_combos([(1, qv, [0]), (-1, [(1,), (-1,)], [0]), (-1, qv, [0])])
    out_qns = ORACLE.zero_flux_combos([(1, qv, [0]), (-1, qv, [0])])
    ab = ORACLE.fill_blocks_normal([(deg[q[0]], 1, deg[q[2]]) for q in a_qns], seed=seed)
    eb = ORACLE.fill_blocks_normal([(deg[q[0]], 1, deg[q[2]]) for q in e_qns], seed=seed + 1)
    return qv, a_qns, ab, e_qns, eb, out_qns


def oracle_c4(seed=777):
    qv, a_qns, ab, e_qns, eb, out_qns = c4_oracle_inputs(seed)
    out, _ = ORACLE.contract_blocks(a_qns, ab, ["vl", "p", "vr"], e_qns, eb, ["vr", "p", "x"], out_qns)
    return out


def cpu_c4(budget_s=3.0):
    qv, a_qns, ab, e_qns, eb, out_qns = c4_oracle_inputs()

    def run():
        ORACLE.zero_flux_combos([(1, qv, [0]), (-1, qv, [0])])
        ORACLE.contract_blocks(a_qns, ab, ["vl", "p", "vr"], e_qns, eb, ["vr", "p", "x"], out_qns)
    best, n = _best_of(run, budget_s, 50)
    return {"value": round(2 * C4_MACS / best / 1e9, 3), "unit": "GFLOP/s", "cores": cpu_threads(), "kind": "port",
            "sample": f"{n} block-sparse contractions (C4), best-of", "ms_per_call": round(best * 1e3, 3)}


def cpu_peps(chi, D, d, n_sites, n_sample=2):
    slots = ORACLE.net_slots(ORACLE.PEPS_NET)
    flop = None
    ts = []
    for s in range(n_sample):
        inp = ORACLE.peps_inputs(chi, D, d, site=s)
        if flop is None:
            sets = {n: ls for n, ls in slots}
            dims = {l: dd for n, ls in slots for l, dd in zip(ls, inp[n].shape)}
            flop = 2 * ORACLE.contraction_cost(ORACLE.find_optimal_order(sets, dims), sets, dims)
        t0 = time.perf_counter()
        ORACLE.launch(slots, "", inp)
        ts.append(time.perf_counter() - t0)
    per = float(np.mean(ts))
    return {"value": round(flop / per / 1e9, 3), "unit": "GFLOP/s", "cores": cpu_threads(), "kind": "port",
            "sample": f"{n_sample} of the {n_sites} sites timed (optimal order each), rate extrapolated "
                      f"linearly to the batch", "s_per_site": round(per, 2)}


def cpu_svd(budget_s=3.0):
    """Oracle port of svd_truncate (np.linalg.svd per sector, same ranking) on the C4
    two-site sector matrices; matricisation excluded (host bookkeeping there)."""
    import paper_2401_01921_b200 as tnb
    psi = c4_two_site(tnb)
    mz = tnb.linalg._Matricized(psi)
    mats = [v[k].cpu().numpy() for m, n, mem, off, v in mz.groups for k in range(len(mem))]
    best, n = _best_of(lambda: ORACLE.svd_truncate_values(mats, 1024), budget_s, 10)
    return {"value": round(best * 1e3, 3), "unit": "ms per svd_truncate", "cores": cpu_threads(), "kind": "port",
            "sample": f"{n} x 23-sector svd_truncate (np.linalg.svd, OpenBLAS), best-of"}


def cpu_utn(path, nbytes, budget_s=2.0):
    best, n = _best_of(lambda: ORACLE.load_utn(path), budget_s, 50)
    return {"value": round(nbytes / best / 1e9, 3), "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"{n} loads of the C4 A tensor into numpy (io.py:83-107 restated), best-of"}


def cpu_lanczos(chi, iters=4):
    """Oracle port of linalg.lanczos with the oracle's L.A.W.R launch as matvec."""
    inp = ORACLE.hermitian_lawr_inputs(chi, seed=7)
    shape = inp["A"].shape

    def mv(v):
        arrs = dict(inp)
        arrs["A"] = v.reshape(shape)
        out, _ = ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", arrs)
        return np.ascontiguousarray(out).reshape(-1)
    t0 = time.perf_counter()
    try:
        ORACLE.lanczos(mv, int(np.prod(shape)), k=1, v0=inp["A"].reshape(-1), tol=1e-14, max_iter=iters, seed=3)
    except RuntimeError:
        pass
    dt = time.perf_counter() - t0
    return {"value": round(dt / iters * 1e3, 3), "unit": "ms per Lanczos iteration", "cores": cpu_threads(),
            "kind": "port", "sample": f"{iters} iterations of the oracle's Lanczos (numpy L.A.W.R matvec, chi={chi})"}


# ----------------------------------------------------------------------------- parity (untimed)
def parity_lawr(out, chi, dtype, seed):
    want, _ = ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", ORACLE.lawr_inputs(chi, dtype=dtype, seed=seed))
    return rel_err(out, want)


def parity_c4(blocks, seed=777):
    want = oracle_c4(seed)
    return rel_err(np.concatenate([b.reshape(-1) for b in blocks]),
                   np.concatenate([w.reshape(-1) for w in want]))


def parity_peps(val, chi, D, d, site=0):
    want, _ = ORACLE.launch(ORACLE.net_slots(ORACLE.PEPS_NET), "", ORACLE.peps_inputs(chi, D, d, site=site))
    return abs(val - float(np.asarray(want).reshape(()))) / abs(float(np.asarray(want).reshape(())))


def parity_permute(samples):
    """Bit-exact check of one permutation per case against np.ascontiguousarray: 0.0 when
    every checked permute is bit-identical, 1.0 otherwise."""
    bad = 0
    for name, shape, dt, p, got in samples:
        src = ORACLE.uniform(list(shape), dtype=dt, seed=11)
        bad += 0 if np.array_equal(got, ORACLE.permute_contiguous(src, p)) else 1
    return float(bad > 0)


# ----------------------------------------------------------------------------- main
def _r(x, nd=4):
    if x is None:
        return None
    if isinstance(x, float):
        return float(f"{x:.{nd}g}")
    return x


def compact(value, unit, frac=None, cpu=None, e2e=None, par=None, ms=None):
    d = {"v": _r(value, 6), "u": unit}
    for k, v in (("frac", frac), ("cpu", cpu), ("e2e", e2e), ("par", par), ("ms", ms)):
        if v is not None:
            d[k] = _r(v, 4 if k != "par" else 2)
    return d


def run_reference(args, dist):
    """--impl reference: the reference algorithm on the host's cores (oracle port)."""
    if dist.rank != 0:
        return 0
    chi = CONFIG["chi"]
    inp = ORACLE.lawr_inputs(chi, dtype=np.float64, seed=1234)
    sets, dims = WL.lawr_label_sets(), WL.lawr_dims(chi)
    tree = ORACLE.find_optimal_order(sets, dims)
    macs, order = ORACLE.contraction_cost(tree, sets, dims), ORACLE.render_order(tree)
    assert order == CONFIG["order"]
    flop = 2 * macs
    for _ in range(args.warmup):
        ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", inp)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", inp)
    dt = (time.perf_counter() - t0) / args.steps
    val = round(flop / dt / 1e9, 3)
    line = {"metric": METRIC, "value": val, "unit": "GFLOP/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA, "config": dict(CONFIG),
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cpu_threads(), "kind": "port",
                             "sample": f"{args.steps} full launches (numpy/OpenBLAS port of tnkit on host cores)"},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "host": host_info()}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tnb", choices=["tnb", "reference"])
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    dist = Dist()
    if args.impl == "reference":
        dist.init("gloo")
        return run_reference(args, dist)

    import torch
    torch.cuda.set_device(dist.local % max(torch.cuda.device_count(), 1))
    dist.init("nccl")
    import paper_2401_01921_b200 as tnb
    flush = L2Flush()
    hbm_peak, hbm_src = peaks()
    cpu_on = dist.rank == 0 and dist.world == 1 and not args.no_cpu
    detail = {}

    with ClockSampler(dist.local) as clk:
        head = gpu_lawr(tnb, 1024, np.float64, args.steps, args.warmup, flush, dist)
    clocks = clk.summary()
    line = {"metric": METRIC, "value": round(head["gflops"], 3), "unit": "GFLOP/s", "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(head["ms_per_step"], 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": dict(CONFIG), "e2e": head["e2e"], "roofline": head["roofline"],
            "gpu_launches": int(head["launches_per_step"] * args.steps), "clocks": clocks,
            "timing": f"L2 flushed per step; CUDA events; max over ranks; replicas x{dist.world}",
            "peak_source": PEAK_SOURCE}
    detail["headline"] = {k: v for k, v in head.items() if k not in ("out", "inp")}
    if dist.rank == 0:
        line["parity"] = {"rel_fro": _r(parity_lawr(head["out"], 1024, np.float64, 1234), 3), "tol": TOL}
    del head
    wl = {}
    if not args.no_secondary:
        only = os.environ.get("TNB_BENCH_ONLY")  # dev: comma-separated subset of workloads

        def w_c1():
            r = gpu_lawr(tnb, 128, np.float64, max(10, args.steps), args.warmup, flush, dist, e2e=True, graph=True,
                         e2e_graph=True)
            detail["C1"] = {k: v for k, v in r.items() if k not in ("out", "inp")}
            cpu = cpu_lawr(128, np.float64, budget_s=2, max_iter=50) if cpu_on else None
            detail["C1"]["cpu_baseline"] = cpu
            par = parity_lawr(r["out"], 128, np.float64, 1234) if dist.rank == 0 else None
            d = compact(r["gflops_graph"], "GFLOP/s", r["roofline"]["frac"], cpu and cpu["value"], r["e2e"]["value"],
                        par, r["graph_ms_per_step"])
            d["v_eager"] = _r(r["gflops"], 5)  # plain Network.launch (host-bound at this size)
            return d

        def w_perm():
            perm, samples = gpu_permute(tnb, max(4, args.steps), args.warmup, flush, dist)
            detail["C2"] = dict(perm)
            med = float(np.median([v["median_gbs"] for v in perm.values()]))
            mn = min(v["min_gbs"] for v in perm.values())
            cpu = cpu_permute() if cpu_on else None
            detail["C2"]["cpu_baseline"] = cpu
            par = parity_permute(samples) if dist.rank == 0 else None
            d = compact(dist.sum(med), "GB/s", med / hbm_peak, cpu and cpu["value"], None, par)
            d["min_frac"] = _r(mn / hbm_peak, 3)
            d["cases_frac"] = {k: _r(v["median_gbs"] / hbm_peak, 3) for k, v in perm.items()}
            return d

        def w_c3():
            r = gpu_lawr(tnb, 1024, np.complex128, max(8, args.steps), args.warmup, flush, dist, e2e=True)
            par = parity_lawr(r["out"], 1024, np.complex128, 1234) if dist.rank == 0 else None
            old = tnb.get_complex_mode()
            try:
                tnb.set_complex_mode("3M")
                r3 = gpu_lawr(tnb, 1024, np.complex128, max(8, args.steps), args.warmup, flush, dist, e2e=False)
                par3 = parity_lawr(r3["out"], 1024, np.complex128, 1234) if dist.rank == 0 else None
            finally:
                tnb.set_complex_mode(old)
            detail["C3_c128"] = {k: v for k, v in r.items() if k not in ("out", "inp")}
            detail["C3_c128"]["3M"] = {k: v for k, v in r3.items() if k not in ("out", "inp")}
            cpu = cpu_lawr(1024, np.complex128, budget_s=3, max_iter=3) if cpu_on else None
            detail["C3_c128"]["cpu_baseline"] = cpu
            d = compact(r["gflops"], "GFLOP/s", r["roofline"]["frac"], cpu and cpu["value"],
                        r["e2e"]["value"], par, r["ms_per_step"])
            d["v_3M"] = _r(r3["gflops"], 6)
            d["par_3M"] = _r(par3, 2)
            return d

        def w_c3b():
            r = gpu_lawr_batch(tnb, 64, 512, np.complex128, max(2, args.steps // 4), 1, flush, dist)
            par = parity_lawr(r["out0"], 512, np.complex128, WL.lawr_batch_seed(0)) if r["out0"] is not None else None
            detail["C3b"] = {k: v for k, v in r.items() if k != "out0"}
            cpu = cpu_lawr_batch(64, 512, np.complex128) if cpu_on else None
            detail["C3b"]["cpu_baseline"] = cpu
            d = compact(r["gflops"], "GFLOP/s", r["roofline"]["frac"], cpu and cpu["value"],
                        r["e2e"]["value"], par, r["ms_per_step"])
            d["scaling"] = "strong"
            return d

        def w_c4():
            r = gpu_c4(tnb, max(10, args.steps), args.warmup, flush, dist)
            par = parity_c4(r.pop("out_blocks")) if dist.rank == 0 else None
            detail["C4"] = r
            cpu = cpu_c4() if cpu_on else None
            detail["C4"]["cpu_baseline"] = cpu
            d = compact(r["gflops"], "GFLOP/s", r["roofline"]["frac"], cpu and cpu["value"],
                        r["e2e"]["value"], par, r["ms_per_call_graph"])
            d["v_eager"] = _r(r["gflops_eager"], 5)
            if "sharded" in r:
                d["v_sharded"] = _r(r["sharded"]["gflops"], 5)
                d["par_sharded"] = _r(r["sharded_par"], 2)
            return d

        def w_c4b():
            r = gpu_c4_batch(tnb, 64, max(3, args.steps // 2), args.warmup, flush, dist)
            out0 = r.pop("out0_blocks")
            par = parity_c4(out0, seed=777) if out0 is not None else None
            detail["C4_batch64"] = r
            d = compact(r["gflops"], "GFLOP/s", r["roofline"]["frac"], None, None, par, r["ms_per_step"])
            d["scaling"] = "strong"
            return d

        def w_peps():
            r = gpu_peps(tnb, 32, 256, 8, 2, 2, 1, flush, dist)
            par = parity_peps(r["site0"], 256, 8, 2) if dist.rank == 0 else None
            detail["C5"] = r
            cpu = cpu_peps(256, 8, 2, 32) if cpu_on else None
            detail["C5"]["cpu_baseline"] = cpu
            d = compact(r["gflops"], "GFLOP/s", r["roofline"]["frac"], cpu and cpu["value"], None, par,
                        r["ms_per_step"])
            d["scaling"] = "strong"
            return d

        def w_svd():
            r = gpu_svd(tnb, 3, 1, flush, dist)
            detail["f3_svd"] = r
            cpu = cpu_svd() if cpu_on else None
            return compact(r["ms_per_call"], "ms/call", None, cpu and cpu["value"])

        def w_lanczos():
            r = gpu_lanczos(tnb, 1024, dist)
            detail["f2_lanczos"] = r
            cpu = cpu_lanczos(1024) if cpu_on else None
            return compact(r["ms_per_iteration"], "ms/iter", None, cpu and cpu["value"])

        def w_utn():
            r = gpu_utn(tnb, 10, 2, dist)
            detail["f4_utn"] = r
            cpu = cpu_utn(r["path"], r["payload_bytes"]) if cpu_on else None
            return compact(r["gbs"], "GB/s (file->HBM)", None, cpu and cpu["value"])

        # each workload is isolated: a failure is recorded, the headline line still prints
        for name, fn in [("C2_permute", w_perm), ("C1_chi128_f64", w_c1), ("C3_chi1024_c128", w_c3),
                         ("C3b_64x_chi512_c128", w_c3b), ("C4_blocksparse", w_c4), ("C4_batch64", w_c4b),
                         ("C5_peps_32sites", w_peps), ("f3_svd", w_svd), ("f2_lanczos", w_lanczos),
                         ("f4_utn", w_utn)]:
            if only and name not in only.split(","):
                continue
            try:
                wl[name] = fn()
            except Exception as e:  # noqa: BLE001
                wl[name] = {"error": f"{type(e).__name__}: {e}"[:200]}
            torch.cuda.empty_cache()
            if cpu_on:
                # a workload's CPU leg leaves 16 OpenBLAS threads spinning for ~0.1 s: they
                # would steal the next workload's host thread (measured: C3 c128 6.09 vs 5.09
                # ms per step right after C1's CPU leg)
                time.sleep(0.5)
        line["workloads"] = wl
        line["workloads_keys"] = "v, frac=roofline, cpu=oracle port, e2e=host buffers, par=rel.err vs oracle, ms/step"
    if cpu_on:
        cb = cpu_lawr(1024, np.float64)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line["host"] = host_info()
    if dist.rank == 0:
        out_dir = os.path.join(ROOT, "gpurun_out")
        if os.path.isdir(out_dir):
            try:
                with open(os.path.join(out_dir, f"bench_detail_n{dist.world}.json"), "w") as f:
                    json.dump({"line": line, "detail": detail}, f, indent=1, default=str)
                line["detail"] = f"gpurun_out/bench_detail_n{dist.world}.json"
            except Exception:
                pass
        print(json.dumps(line, separators=(",", ":")), flush=True)
    return 0


import tnkit_np as ORACLE  # noqa: E402  (checker, CPU-baseline leg and reference arm only)
from paper_2401_01921_b200 import workloads as WL  # noqa: E402

if __name__ == "__main__":
    sys.exit(main())

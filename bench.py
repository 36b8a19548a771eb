"""Benchmark driver (contract: README of the round / SURVEY.md section 8(d)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tnb|reference]
                    [--workload NAME] [--no-secondary]

Headline workload (BASELINE.json configs[2], f64 part, the north-star target):
L.A.W.R effective-Hamiltonian matvec through ``Network.launch`` at chi=1024, d=2,
D=5, float64, optimal order (((A,L),W),R); metric fp64 GFLOP/s (algorithmic
2*MACs from the reference's own cost model). Secondary workloads (configs C1,
C2, C3 c128 / batch, C4, C5) are measured in the same run and reported under
"workloads". Inputs are the reference recipes' seeded N(0,1)/U(0,1) synthetic
tensors (oracle/tnkit_np.py) -- there is no dataset.

--impl reference times the reference algorithm's CPU path (the numpy port in
oracle/, same numpy/OpenBLAS calls as the reference) on this host's cores.
Multi-GPU (torchrun): one process per GPU; the matvec is replicated per rank
(weak scaling), the C3b batch and C5 sites are sharded across ranks.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np

FP64_PEAK_TFLOPS = 37.06   # measured DMMA peak on this pool's B200 (profiles/r01_fp64_peak.txt)
PEAK_SOURCE = "measured DMMA.8x8x4 microbenchmark, profiles/r01_fp64_peak.txt (MEASURED_PEAKS.json has no fp64)"


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
    capture of this workload (profiles/r01_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            tr = json.load(f)
        key = f"{kernel}:{np.dtype(dtype).name}"
        return tr[key]["bytes_per_launch"] if key in tr else None
    except Exception:
        return None


# ----------------------------------------------------------------------------- dist
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, backend):
        if self.world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            import torch
            if torch.cuda.is_available():
                self.pg.barrier(device_ids=[self.local])
            else:
                self.pg.barrier()

    def max(self, x):
        if not self.pg:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64,
                         device="cuda" if torch.cuda.is_available() else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x):
        if not self.pg:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64,
                         device="cuda" if torch.cuda.is_available() else "cpu")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())


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


# ----------------------------------------------------------------------------- GPU side
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


def time_steps(fn, steps, flush, dist):
    """Device time of `steps` calls of fn, each bracketed by its own events; L2 flushed
    (untimed) before every call; barrier + synchronize around the region; max over ranks.
    Python's cyclic GC is collected before and paused during the region (as timeit does): a
    generation-2 pass over a large heap is a 10-40 ms host stall unrelated to the work."""
    import gc
    import torch
    pairs = []
    dist.barrier()
    gc.collect()
    torch.cuda.synchronize()
    was = gc.isenabled()
    gc.disable()
    try:
        for _ in range(steps):
            flush()
            e0, e1 = _events()
            e0.record()
            fn()
            e1.record()
            pairs.append((e0, e1))
        torch.cuda.synchronize()
    finally:
        if was:
            gc.enable()
    dist.barrier()
    total_ms = sum(a.elapsed_time(b) for a, b in pairs)
    return dist.max(total_ms)


def lawr_network(tnb, inp):
    net = tnb.Network(WL.LAWR_NET)
    tensors = {}
    for nm, arr in inp.items():
        t = tnb.UniTensor(tnb.storage.from_numpy(arr), labels=[f"{nm}{i}" for i in range(arr.ndim)])
        net.put_tensor(nm, t, t.labels)
        tensors[nm] = t
    net.set_order(optimal=True)
    return net, tensors


def lawr_macs(chi, d=2, D=5):
    import paper_2401_01921_b200 as tnb
    sets, dims = WL.lawr_label_sets(), WL.lawr_dims(chi, d, D)
    tree = tnb.find_optimal_order(sets, dims)
    return tnb.contraction_cost(tree, sets, dims), tnb.render_order(tree)


E2E_CHUNKS = int(os.environ.get("TNB_E2E_CHUNKS", "2"))  # 1-8 swept with double buffering: 2 best


def gpu_lawr(tnb, chi, dtype, steps, warmup, flush, dist, e2e=True, roof=True, seed=1234, graph=False):
    import torch
    inp = WL.lawr_inputs(chi, dtype=dtype, seed=seed + 17 * dist.rank)
    net, tensors = lawr_network(tnb, inp)
    macs, order = lawr_macs(chi)
    flop = macs * (8 if dtype == np.complex128 else 2)
    for _ in range(warmup):
        net.launch()
    launches0 = tnb._lib.launch_count()
    ms = time_steps(net.launch, steps, flush, dist)
    launches = (tnb._lib.launch_count() - launches0) // max(steps, 1)
    assert net.get_order() == order
    res = {"ms_per_step": ms / steps, "flop_per_step": flop, "order": order, "launches_per_step": launches}
    res["gflops"] = dist.sum(flop) / (ms / steps) / 1e6  # all ranks' work / max time
    if graph:
        # the same launch replayed from Network.compile() (CUDA graph: no host work per step)
        cn = net.compile()
        for _ in range(warmup):
            cn.launch()
        gms = time_steps(cn.launch, steps, flush, dist) / steps
        res["graph_ms_per_step"] = gms
        res["gflops_graph"] = dist.sum(flop) / gms / 1e6
    if e2e:
        # end to end through the public API: pinned host inputs -> HBM, launch, result -> host.
        # A serving loop: two networks with their own device inputs and pinned host
        # buffers alternate (double buffering), so step i+1's uploads -- each ordered only
        # after the launch that last read that buffer set (upload_(after=net.done_event)) --
        # overlap step i's kernels; every step still copies all of its inputs in and its
        # result out.
        sets = [(net, tensors)] + [lawr_network(tnb, inp)]
        pinned = [{nm: torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for nm, a in inp.items()}
                  for _ in sets]
        h2d = sum(p.numel() * p.element_size() for p in pinned[0].values())
        probe = net.launch().get_block_().contiguous().storage()
        outs = [torch.empty(probe.shape, dtype=probe.dtype, pin_memory=True) for _ in sets]

        # uploads in first-use order on the engine's copy stream: each contraction step
        # waits only for its own operands (and chunk by chunk for chunked ones), so R's copy
        # runs under the A.L GEMM and the T2.R GEMM trails R's upload panel by panel
        first_use = tnb.tree_leaves(tnb.parse_order(order))

        def step(i):
            n, ts = sets[i % 2]
            for nm in first_use:
                # large operands in chunks: each contraction step that consumes one runs its
                # column panels as the chunks land (upload and GEMM overlap)
                big = pinned[0][nm].numel() * pinned[0][nm].element_size() >= (8 << 20)
                ts[nm].get_block_().upload_(pinned[i % 2][nm], chunks=E2E_CHUNKS if big else 1, after=n.done_event)
            n.launch(host_out=outs[i % 2])  # result streamed to the pinned host buffer

        def run(k):
            import gc
            dist.barrier()
            gc.collect()
            torch.cuda.synchronize()
            gc.disable()  # as in time_steps
            try:
                e0, e1 = _events()
                e0.record()
                for i in range(k):
                    step(i)
                e1.record()
                torch.cuda.synchronize()
            finally:
                gc.enable()
            dist.barrier()
            return dist.max(e0.elapsed_time(e1))
        run(max(2, warmup))
        ems = run(steps)
        lat = run(1)  # one step alone: latency, no overlap with a neighbour
        d2h = outs[0].numel() * outs[0].element_size()
        res["e2e"] = {"value": dist.sum(flop) / (ems / steps) / 1e6, "unit": "GFLOP/s",
                      "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                      "ms_per_step": ems / steps, "single_step_latency_ms": lat,
                      "pipelining": "double-buffered inputs/outputs, upload of step i+1 overlaps step i"}
    if roof:
        # dominant kernel = the stream-K DMMA GEMM (steps A.L and T2.R): the library's kernel
        # timer records a CUDA event pair around each of its launches ON THE LAUNCHING STREAM;
        # this pass repeats the timed region (same flush, same K steps) with the timer on.
        tnb._lib.ktimer_reset()
        tnb._lib.ktimer_enable(True)
        time_steps(net.launch, steps, flush, dist)
        tnb._lib.ktimer_enable(False)
        n_g, ms_g, fl_g = tnb._lib.ktimer_read(tnb._lib.KF_GEMM)
        n_s, ms_s, _ = tnb._lib.ktimer_read(tnb._lib.KF_GEMM_SKINNY)
        tnb._lib.ktimer_reset()
        ach = fl_g / (dist.max(ms_g) / 1e3) / 1e12 if n_g else 0.0  # per GPU (slowest rank)
        res["steps_ms"] = {"gemm (A.L + T2.R)": ms_g / steps, "skinny (T1.W)": ms_s / steps,
                           "gemm_launches_per_step": n_g / steps, "gemm_share_of_step": ms_g / ms}
        res["roofline"] = {"bound": "tensor", "achieved": round(ach, 3), "peak": FP64_PEAK_TFLOPS,
                           "unit": "TFLOP/s", "frac": round(ach / FP64_PEAK_TFLOPS, 4),
                           "traffic": traffic_per_launch("gemm_sk_kernel", dtype),
                           "kernel": "gemm_sk_kernel (stream-K DMMA.8x8x4), steps A.L + T2.R",
                           "achieved_how": "algorithmic flop of the GEMM launches / their summed CUDA-event "
                                           "durations on the launching stream, over the K timed steps",
                           "peak_source": PEAK_SOURCE}
    return res


def gpu_permute(tnb, steps, warmup, flush, dist):
    import itertools
    import torch
    out = {}
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
        rates, eager = [], []
        k = max(1, steps // 2)
        for p in perms:
            for _ in range(warmup):
                src.permute(*p).contiguous()
            ms = time_steps(lambda: src.permute(*p).contiguous(), k, flush, dist) / k
            eager.append(nbytes / ms / 1e6)
            # device time: the same call replayed from a CUDA graph (no host work in the window)
            g = tnb.graphs.capture(lambda: src.permute(*p).contiguous(), warmup=1)
            gms = time_steps(g.replay, k, flush, dist) / k
            rates.append(nbytes / gms / 1e6)
            del g
        out[name] = {"median_gbs": float(np.median(rates)), "min_gbs": float(np.min(rates)),
                     "max_gbs": float(np.max(rates)), "eager_median_gbs": float(np.median(eager)),
                     "n_perms": len(perms), "bytes_per_permute": nbytes}
    return out


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
    import torch
    A, E = c4_tensors(tnb)
    for _ in range(warmup):
        tnb.contract(A, E)
    ms = time_steps(lambda: tnb.contract(A, E), steps, flush, dist) / steps
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        tnb.contract(A, E)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / steps * 1e3
    # device time of the same call replayed as a CUDA graph (plan cached on device)
    g = tnb.graphs.capture(lambda: tnb.contract(A, E))
    gms = time_steps(g.replay, steps, flush, dist) / steps
    tnb._lib.ktimer_reset()
    tnb._lib.ktimer_enable(True)
    time_steps(lambda: tnb.contract(A, E), steps, flush, dist)
    tnb._lib.ktimer_enable(False)
    n_k, ms_k, _ = tnb._lib.ktimer_read(tnb._lib.KF_BS_GEMM)
    tnb._lib.ktimer_reset()
    kms = ms_k / max(n_k, 1)
    extra = {}
    if dist.world > 1:
        # one C4 contraction partitioned over the ranks (LPT output panels, local K
        # reduction, NCCL all-gather of the slab): strong scaling of a single call
        from paper_2401_01921_b200 import parallel
        for _ in range(warmup):
            parallel.contract_sharded(A, E)
        sms = time_steps(lambda: parallel.contract_sharded(A, E), steps, flush, dist) / steps
        extra = {"sharded_ms_per_call": sms, "sharded_gflops": 2 * C4_MACS / sms / 1e6,
                 "sharded_scaling": "strong (one contraction partitioned over ranks + NCCL all-gather)"}
    return {**extra, "ms_per_call_eager": ms, "host_wall_ms_per_call": wall, "ms_per_call_graph": gms,
            "bs_gemm_kernel_ms": kms, "bs_gemm_kernel_tflops": 2 * C4_MACS / kms / 1e9,
            "gflops_eager": dist.sum(2 * C4_MACS) / ms / 1e6, "gflops": dist.sum(2 * C4_MACS) / gms / 1e6}


def gpu_c4_batch(tnb, n_total, steps, warmup, flush, dist):
    """A batch of independent C4 block-sparse contractions (e.g. the sites of a sweep),
    sharded by unit across ranks (no data-path collective): strong scaling of the batch."""
    mine = [i for i in range(n_total) if i % dist.world == dist.rank]
    pairs = [c4_tensors(tnb, seed=777 + 2 * i) for i in mine]

    def step():  # one grouped launch over the output tiles of all of this rank's contractions
        tnb.contract_batched(pairs)

    def step_pairwise():
        for A, E in pairs:
            tnb.contract(A, E)
    for _ in range(warmup):
        step()
    ms = time_steps(step, steps, flush, dist) / steps
    for _ in range(warmup):
        step_pairwise()
    ms_pw = time_steps(step_pairwise, steps, flush, dist) / steps
    tnb._lib.ktimer_reset()
    tnb._lib.ktimer_enable(True)
    time_steps(step, steps, flush, dist)
    tnb._lib.ktimer_enable(False)
    n_k, ms_k, _ = tnb._lib.ktimer_read(tnb._lib.KF_BS_GEMM)
    tnb._lib.ktimer_reset()
    kms = dist.max(ms_k / max(steps, 1))
    return {"ms_per_step": ms, "instances": n_total, "per_rank": len(mine),
            "gflops": 2 * C4_MACS * n_total / ms / 1e6, "api": "contract_batched (tnb_bs_execute_batched)",
            "bs_gemm_kernel_ms": kms, "bs_gemm_kernel_tflops": 2 * C4_MACS * len(mine) / kms / 1e9 if kms else 0.0,
            "ms_per_step_pairwise": ms_pw, "gflops_pairwise": 2 * C4_MACS * n_total / ms_pw / 1e6}


def gpu_lawr_batch(tnb, n_total, chi, dtype, steps, warmup, flush, dist):
    """C3b: a batch of independent L.A.W.R matvecs, sharded by instance across ranks."""
    mine = [i for i in range(n_total) if i % dist.world == dist.rank]
    nets = []
    for i in mine:
        net, _ = lawr_network(tnb, WL.lawr_inputs(chi, dtype=dtype, seed=5000 + 4 * i))
        nets.append(net)
    macs, _ = lawr_macs(chi)
    flop = macs * (8 if dtype == np.complex128 else 2)

    def step():
        for net in nets:
            net.launch()
    for _ in range(warmup):
        step()
    ms = time_steps(step, steps, flush, dist) / steps
    return {"ms_per_step": ms, "instances": n_total, "per_rank": len(mine),
            "gflops": flop * n_total / ms / 1e6}


def gpu_peps(tnb, n_sites, chi, D, d, steps, warmup, flush, dist):
    """C5 (reading A): PEPS double-layer site networks, optimal order, sharded by site."""
    mine = [i for i in range(n_sites) if i % dist.world == dist.rank]
    shapes = WL.peps_shapes(chi, D, d)
    net = tnb.Network(WL.PEPS_NET)
    tensors = {}
    for k, (nm, shp) in enumerate(shapes.items()):
        t = tnb.UniTensor(tnb.storage.from_numpy(tnb.storage.host_normal(shp, seed=9000 + k)),
                          labels=[f"x{j}" for j in range(len(shp))])
        net.put_tensor(nm, t)
        tensors[nm] = t
    net.set_order(optimal=True)
    sets = {n: ls for n, ls in net._slots}
    dims = {}
    for nm, ls in net._slots:
        for l, dd in zip(ls, shapes[nm]):
            dims[l] = dd
    tree = tnb.find_optimal_order(sets, dims)
    flop = 2 * tnb.contraction_cost(tree, sets, dims)

    def step():
        for _ in mine:  # every site re-launches the blueprint (inputs differ per site in a real sweep)
            net.launch()
    for _ in range(max(1, warmup)):
        net.launch()
    ms = time_steps(step, steps, flush, dist) / steps
    return {"ms_per_step": ms, "sites": n_sites, "per_rank": len(mine), "order": tnb.render_order(tree),
            "flop_per_site": flop, "gflops": flop * n_sites / ms / 1e6}


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
    import torch
    psi = c4_two_site(tnb)
    fn = lambda: tnb.linalg.svd_truncate(psi, keepdim=1024)  # noqa: E731
    for _ in range(max(1, warmup)):
        fn()
    ms = time_steps(fn, steps, flush, dist) / steps
    return {"ms_per_call": ms, "keepdim": 1024, "sectors": 23,
            "note": "float64 sectors: one launch of the batched one-sided Jacobi kernel (tnb_svd_jacobi_batched, "
                    "a 16-CTA cluster per sector); matricise/scatter = tnb_copy2d_batched"}


LANCZOS_ITERS = 30


def gpu_lanczos(tnb, chi, dist):
    """(f)1+(f)2 workload: Lanczos iterations on the Hermitian L.A.W.R effective Hamiltonian
    at chi (ORACLE.hermitian_lawr_inputs), matvec = the compiled Network replayed as a CUDA
    graph, Krylov basis + full reorthogonalisation in HBM. Fixed iteration count
    (max_iter) so GPU and CPU time the same work: ms per Lanczos iteration."""
    import torch
    from paper_2401_01921_b200 import eig
    inp = ORACLE.hermitian_lawr_inputs(chi, seed=7)
    net, _ = lawr_network(tnb, inp)
    op = eig.NetworkMatvec(net.compile(), "A")
    v0 = torch.from_numpy(np.ascontiguousarray(inp["A"]).reshape(-1)).cuda()  # DMRG: start from psi

    def run():
        try:
            eig.lanczos(op, k=1, v0=v0, tol=1e-14, max_iter=LANCZOS_ITERS, seed=3)
        except eig.ConvergenceError:
            pass
    run()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    run()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    return {"ms_per_iteration": ms / LANCZOS_ITERS, "iterations": LANCZOS_ITERS, "chi": chi,
            "matvec": "Network.compile() graph replay (L.A.W.R, f64)"}


def gpu_utn(tnb, steps, warmup, dist):
    """(f)4 workload: .utn load of the C4 MPS tensor A (6.1 MB payload) from the page cache
    into HBM (host wall: read + one H2D + one scatter launch, synchronised)."""
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


def cpu_lawr(chi, dtype, budget_s=8.0, max_iter=10, seed=1234):
    inp = ORACLE.lawr_inputs(chi, dtype=dtype, seed=seed)
    sets, dims = WL.lawr_label_sets(), WL.lawr_dims(chi)
    macs = ORACLE.contraction_cost(ORACLE.find_optimal_order(sets, dims), sets, dims)
    flop = macs * (8 if dtype == np.complex128 else 2)
    ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", inp)  # warm
    ts = []
    t_start = time.perf_counter()
    while len(ts) < max_iter and (time.perf_counter() - t_start) < budget_s:
        t0 = time.perf_counter()
        ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", inp)
        ts.append(time.perf_counter() - t0)
    best = min(ts)
    return {"value": flop / best / 1e9, "unit": "GFLOP/s", "cores": cpu_threads(), "kind": "port",
            "sample": f"{len(ts)} Network launches of L.A.W.R chi={chi} {np.dtype(dtype).name} "
                      f"(oracle port of tnkit, numpy {np.__version__} OpenBLAS), best-of",
            "ms_per_launch": best * 1e3}


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
    return {"value": float(np.median(rates)), "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"{len(rates)} of the 23 rank-4 [64]^4 f64 permutes (np.ascontiguousarray, single-threaded)"}


def cpu_svd(budget_s=3.0):
    """Oracle port of svd_truncate (np.linalg.svd per sector, same ranking) on the C4
    two-site sector matrices; matricisation excluded (it is host bookkeeping there)."""
    import torch
    import paper_2401_01921_b200 as tnb
    psi = c4_two_site(tnb)
    mz = tnb.linalg._Matricized(psi)
    mats = [v[k].cpu().numpy() for m, n, mem, off, v in mz.groups for k in range(len(mem))]
    ts = []
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s and len(ts) < 10:
        t0 = time.perf_counter()
        ORACLE.svd_truncate_values(mats, 1024)
        ts.append(time.perf_counter() - t0)
    return {"value": min(ts) * 1e3, "unit": "ms per svd_truncate", "cores": cpu_threads(), "kind": "port",
            "sample": f"{len(ts)} x 23-sector svd_truncate (np.linalg.svd, OpenBLAS), best-of"}


def cpu_utn(path, nbytes, budget_s=2.0):
    ts = []
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s and len(ts) < 50:
        t0 = time.perf_counter()
        ORACLE.load_utn(path)
        ts.append(time.perf_counter() - t0)
    best = min(ts)
    return {"value": nbytes / best / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"{len(ts)} loads of the C4 A tensor into numpy (io.py:83-107 restated), best-of",
            "ms_per_load": best * 1e3}


def cpu_lanczos(chi, iters=4):
    """Oracle port of linalg.lanczos with the oracle's L.A.W.R launch as matvec (the
    reference's DMRG inner loop on numpy/OpenBLAS), `iters` iterations."""
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
    return {"value": dt / iters * 1e3, "unit": "ms per Lanczos iteration", "cores": cpu_threads(), "kind": "port",
            "sample": f"{iters} iterations of the oracle's Lanczos (numpy L.A.W.R matvec, chi={chi})"}


def cpu_c4(budget_s=3.0):
    sec = ORACLE.c4_sectors()
    qv = [(q,) for q, _ in sec]
    deg = [d for _, d in sec]
    a_qns = ORACLE.zero_flux_combos([(1, qv, [0]), (1, [(1,), (-1,)], [0]), (-1, qv, [0])])
    e_qns = ORACLE.zero_flux_combos([(1, qv, [0]), (-1, [(1,), (-1,)], [0]), (-1, qv, [0])])
    out_qns = ORACLE.zero_flux_combos([(1, qv, [0]), (-1, qv, [0])])
    ab = ORACLE.fill_blocks_normal([(deg[q[0]], 1, deg[q[2]]) for q in a_qns], seed=777)
    eb = ORACLE.fill_blocks_normal([(deg[q[0]], 1, deg[q[2]]) for q in e_qns], seed=778)
    ts = []
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s and len(ts) < 50:
        t0 = time.perf_counter()
        ORACLE.zero_flux_combos([(1, qv, [0]), (-1, qv, [0])])
        ORACLE.contract_blocks(a_qns, ab, ["vl", "p", "vr"], e_qns, eb, ["vr", "p", "x"], out_qns)
        ts.append(time.perf_counter() - t0)
    best = min(ts)
    return {"value": 2 * C4_MACS / best / 1e9, "unit": "GFLOP/s", "cores": cpu_threads(), "kind": "port",
            "sample": f"{len(ts)} block-sparse contractions (C4), best-of", "ms_per_call": best * 1e3}


# ----------------------------------------------------------------------------- main
def run_reference(args, dist):
    """--impl reference: the reference algorithm on the host's cores (oracle port)."""
    if dist.rank != 0:
        return 0
    chi = 1024
    inp = ORACLE.lawr_inputs(chi, dtype=np.float64, seed=1234)
    sets, dims = WL.lawr_label_sets(), WL.lawr_dims(chi)
    tree = ORACLE.find_optimal_order(sets, dims)
    macs, order = ORACLE.contraction_cost(tree, sets, dims), ORACLE.render_order(tree)
    flop = 2 * macs
    for _ in range(args.warmup):
        ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", inp)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ORACLE.launch(ORACLE.lawr_slots(), "b, q, b2", inp)
    dt = (time.perf_counter() - t0) / args.steps
    val = flop / dt / 1e9
    line = {"metric": "fp64 GFLOP/s (L.A.W.R Network matvec, chi=1024)", "value": round(val, 3),
            "unit": "GFLOP/s", "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded N(0,1), reference recipe)",
            "config": {"workload": "lawr_f64_chi1024", "chi": chi, "d": 2, "D": 5, "order": order},
            "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": cpu_threads(), "kind": "port",
                             "sample": f"{args.steps} full launches (numpy/OpenBLAS port of tnkit on host cores)"},
            "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
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
    dist = Dist()
    if args.impl == "reference":
        dist.init("gloo")
        return run_reference(args, dist)

    import torch
    torch.cuda.set_device(dist.local)
    dist.init("nccl")
    import paper_2401_01921_b200 as tnb
    flush = L2Flush()
    hbm_peak, hbm_src = peaks()

    with ClockSampler(dist.local) as clk:
        head = gpu_lawr(tnb, 1024, np.float64, args.steps, args.warmup, flush, dist)
    clocks = clk.summary()
    line = {"metric": "fp64 GFLOP/s (L.A.W.R Network matvec, chi=1024)", "value": round(head["gflops"], 3),
            "unit": "GFLOP/s", "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(head["ms_per_step"], 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded N(0,1), reference recipe)",
            "config": {"workload": "lawr_f64_chi1024", "chi": 1024, "d": 2, "D": 5, "order": head["order"],
                       "l2": "flushed before every timed step (256 MiB write + 256 MiB read, untimed)",
                       "python_gc": "collected before, paused during timed regions (as timeit)", "parallelism":
                       f"replicas x{dist.world}"},
            "e2e": {k: (round(v, 4) if isinstance(v, float) else v) for k, v in head["e2e"].items()},
            "roofline": head["roofline"], "gpu_launches": int(head["launches_per_step"] * args.steps),
            "clocks": clocks, "steps_ms": head["steps_ms"]}
    if not args.no_secondary:
        wl = {}

        def w_c3():
            c3 = gpu_lawr(tnb, 1024, np.complex128, max(3, args.steps // 2), args.warmup, flush, dist, e2e=False)
            res = {"value": round(c3["gflops"], 2), "unit": "GFLOP/s (8 flop/complex MAC)",
                   "ms_per_step": c3["ms_per_step"], "roofline": c3["roofline"], "complex_mode": tnb.get_complex_mode()}
            # the Gauss / 3M formulation (3 real products per complex MAC; same 1e-12 parity tests)
            old = tnb.get_complex_mode()
            try:
                tnb.set_complex_mode("3M")
                c3m = gpu_lawr(tnb, 1024, np.complex128, max(3, args.steps // 2), args.warmup, flush, dist,
                               e2e=False, roof=False)
                res["value_3M"] = round(c3m["gflops"], 2)
                res["ms_per_step_3M"] = c3m["ms_per_step"]
            finally:
                tnb.set_complex_mode(old)
            return res

        def w_c1():
            c1 = gpu_lawr(tnb, 128, np.float64, max(10, args.steps), args.warmup, flush, dist, e2e=False, roof=False,
                          graph=True)
            return {"value": round(c1["gflops"], 2), "unit": "GFLOP/s (eager Network.launch)",
                    "ms_per_step": c1["ms_per_step"], "graph_ms_per_step": c1["graph_ms_per_step"],
                    "gflops_graph": round(c1["gflops_graph"], 2)}

        def w_perm():
            perm = gpu_permute(tnb, max(4, args.steps), args.warmup, flush, dist)
            return {"unit": "GB/s (2 x bytes / time, median over perms)", "cases": perm,
                    "roofline": {"bound": "hbm", "peak": hbm_peak, "unit": "GB/s", "peak_source": hbm_src,
                                 "frac_median": {k: round(v["median_gbs"] / hbm_peak, 4) for k, v in perm.items()}}}

        def w_c4():
            c4 = gpu_c4(tnb, max(10, args.steps), args.warmup, flush, dist)
            return {"value": round(c4["gflops"], 2), "unit": "GFLOP/s (graph replay; eager in gflops_eager)", **c4,
                    "roofline": {"bound": "tensor", "achieved": round(c4["bs_gemm_kernel_tflops"], 3),
                                 "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                                 "frac": round(c4["bs_gemm_kernel_tflops"] / FP64_PEAK_TFLOPS, 4),
                                 "traffic": traffic_per_launch("bs_sk_kernel", np.float64),
                                 "kernel": "bs_sk_kernel (grouped stream-K DMMA.8x8x4)", "peak_source": PEAK_SOURCE}}

        def w_c4b():
            cb = gpu_c4_batch(tnb, 64, max(3, args.steps // 2), args.warmup, flush, dist)
            return {"value": round(cb["gflops"], 2), "unit": "GFLOP/s",
                    "scaling": "strong (64 contractions sharded over ranks)", **cb,
                    "roofline": {"bound": "tensor", "achieved": round(cb["bs_gemm_kernel_tflops"], 3),
                                 "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                                 "frac": round(cb["bs_gemm_kernel_tflops"] / FP64_PEAK_TFLOPS, 4),
                                 "kernel": "bs_sk_kernel, batched (one launch per rank)", "peak_source": PEAK_SOURCE}}

        def w_c3b():
            bt = gpu_lawr_batch(tnb, 64, 512, np.complex128, max(2, args.steps // 4), 1, flush, dist)
            return {"value": round(bt["gflops"], 2), "unit": "GFLOP/s (8 flop/complex MAC)",
                    "scaling": "strong (64 instances sharded over ranks)", **bt}

        def w_peps():
            pe = gpu_peps(tnb, 32, 256, 8, 2, 1, 1, flush, dist)
            return {"value": round(pe["gflops"], 2), "unit": "GFLOP/s", "scaling": "strong (32 sites sharded over ranks)",
                    **pe}

        def w_svd():
            sv = gpu_svd(tnb, 3, 1, flush, dist)
            return {"value": round(sv["ms_per_call"], 3), "unit": "ms per call", "higher_is_better": False, **sv}

        def w_lanczos():
            lz = gpu_lanczos(tnb, 1024, dist)
            return {"value": round(lz["ms_per_iteration"], 4), "unit": "ms per Lanczos iteration",
                    "higher_is_better": False, **lz}

        def w_utn():
            ut = gpu_utn(tnb, 10, 2, dist)
            return {"value": round(ut["gbs"], 3), "unit": "GB/s (payload / host wall)", **ut}

        # each secondary workload is isolated: a failure is recorded, the headline line still prints
        for name, fn in [("permute_sweep", w_perm), ("lawr_c128_chi1024", w_c3), ("lawr_f64_chi128", w_c1),
                         ("blocksparse_c4", w_c4), ("blocksparse_c4_batch64", w_c4b),
                         ("lawr_batch64_c128_chi512", w_c3b), ("peps_chi256_D8", w_peps),
                         ("svd_truncate_two_site_c4", w_svd), ("lanczos_lawr_chi1024", w_lanczos),
                         ("utn_load_c4", w_utn)]:
            only = os.environ.get("TNB_BENCH_ONLY")  # dev: comma-separated subset of secondary workloads
            if only and name not in only.split(","):
                continue
            try:
                wl[name] = fn()
            except Exception as e:  # noqa: BLE001
                wl[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
        line["workloads"] = wl
    if dist.rank == 0 and not args.no_cpu:
        cb = cpu_lawr(1024, np.float64)
        line["cpu_baseline"] = cb
        if not args.no_secondary:
            wl = line["workloads"]
            cpu_legs = [("lawr_f64_chi128", lambda: cpu_lawr(128, np.float64, budget_s=2, max_iter=50)),
                        ("permute_sweep", cpu_permute), ("blocksparse_c4", cpu_c4),
                        ("svd_truncate_two_site_c4", cpu_svd), ("lanczos_lawr_chi1024", lambda: cpu_lanczos(1024)),
                        ("utn_load_c4", lambda: cpu_utn(wl["utn_load_c4"]["path"], wl["utn_load_c4"]["payload_bytes"]))]
            for name, fn in cpu_legs:
                if name in wl and "error" not in wl[name]:
                    try:
                        wl[name]["cpu_baseline"] = fn()
                    except Exception as e:  # noqa: BLE001
                        wl[name]["cpu_baseline"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if dist.rank == 0:
        print(json.dumps(line))
    return 0


import tnkit_np as ORACLE  # noqa: E402  (CPU-baseline leg and reference arm only)
from paper_2401_01921_b200 import workloads as WL  # noqa: E402

if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 DFA-minimization engine.

Metric (BASELINE.json): transitions refined per second (n*k*passes / wall time)
and wall time to the minimal DFA.  A "step" is one complete minimization of
one synthetic DFA to its canonical minimal partition (all refinement passes +
canonical relabel), DFA resident in HBM before the timed region.

Default workload (N=1): the north-star single-GPU configuration — sortPR on
random_dfa(n=1e8, k=4, seed=1, p=0.5) (SURVEY.md §8(d) C5 / BASELINE.md §4),
generated on the device bit-exactly with the reference generator.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)

Multi-GPU (N > 1): one random_dfa of N x 1e8 states, state-sharded over the N
ranks (paper_2410_22764_b200/sharded.py: NCCL all-gather of block ids + key
all-to-all per pass; weak scaling, 1e8 states per GPU); timing is the max over
ranks.  --replicas runs N independent single-GPU minimizations instead.

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified dfamin headers) on the host cores, on a bounded sample of the same
workload; rank 0 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "transitions refined/s to the minimal DFA (n*k*passes / wall time)"
UNIT = "transitions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--algo", default="sort",
                    choices=["sort", "naive", "transpr", "naive_cas", "trans"])
    ap.add_argument("--family", default="random",
                    choices=["random", "chain", "comb", "fib", "bits", "vlts"],
                    help="random: random_dfa(n,k,seed,p); chain: chain_dfa(n); comb: comb(n,3); "
                         "fib: fib_dfa(n) (word index); bits: bit_splitter(n); "
                         "vlts: inflated VLTS-shaped (m=--vlts-m, n, k)")
    ap.add_argument("--vlts-m", type=int, default=1000)
    ap.add_argument("--n", type=int, default=100_000_000)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--p", type=float, default=0.5)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--sortpr-engine", default="hash", choices=["hash", "radix"])
    ap.add_argument("--cpu-sample-n", type=int, default=10_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas instead of the state-sharded sortPR")
    ap.add_argument("--sharded", action="store_true",
                    help="run the state-sharded sortPR driver even at N = 1 (its own baseline)")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def int8_peak():
    """Dense int8 tensor peak.  The measured cuBLASLt int8 GEMM (profiles/int8_peak.json,
    3.09 POP/s) is slower than this repo's own tcgen05 kind::i8 squaring, so it is no
    ceiling: the roofline uses the nominal dense B200 int8 peak, 4.5 POP/s."""
    return 4500.0, "nominal dense int8 (4.5 POP/s; cuBLASLt int8 measured 3.09 POP/s, " \
                    "profiles/int8_peak.json)"


# the workloads profiles/ncu_traffic.json was captured on: (family, algo, n, k)
TRAFFIC_WORKLOAD = {"gemm": ("fib", "trans", 12, 1)}
TRAFFIC_DEFAULT = ("random", "sort", 100_000_000, 4)


def ncu_traffic(family: str, args=None):
    """dram bytes per step for a kernel family from the committed ncu summary, or
    None when this run is not the workload that summary was captured on."""
    if args is not None and (args.family, args.algo, args.n, args.k) != \
            TRAFFIC_WORKLOAD.get(family, TRAFFIC_DEFAULT):
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(family)
    except Exception:
        return None


# ----------------------------------------------------------------- CPU baseline
def cpu_reference_sample(n: int, k: int, seed: int, p: float, threads: int, steps: int = 1):
    """The unmodified reference sort_pr (oracle/_ref) on host cores; returns
    (transitions/s per step list, iterations, kind, sample, cores)."""
    import numpy as np
    import paper_2410_22764_b200 as dfm
    from oracle import oracle as O
    d = dfm.random_dfa(n, k, seed, p)  # bit-exact with generators.hpp:130-145
    if O.ref_available():
        R = O.Reference()
        R.set_threads(threads)
        runs = []
        for _ in range(steps):
            r = R.sort_pr(d.delta, d.accepting)
            runs.append((n * k * r.iterations) / (r.elapsed_ms / 1e3))
        return runs, r.iterations, "reference", R.worker_count(), r.elapsed_ms
    # oracle port (plain C restatement, single-threaded)
    runs = []
    for _ in range(steps):
        t0 = time.perf_counter()
        r = O.sort_pr(d.delta, d.accepting)
        dt = time.perf_counter() - t0
        runs.append((n * k * r.iterations) / dt)
    return runs, r.iterations, "port", 1, dt * 1e3


def run_reference_arm(args, rank: int, world: int):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n = min(args.n, args.cpu_sample_n)
    t_all = time.perf_counter()
    for _ in range(args.warmup):
        cpu_reference_sample(n, args.k, args.seed, args.p, threads)
    vals = []
    iters = None
    kind = cores = None
    ms = []
    for _ in range(args.steps):
        v, iters, kind, cores, el = cpu_reference_sample(n, args.k, args.seed, args.p, threads)
        vals.append(v[0])
        ms.append(el)
    value = statistics.mean(vals)
    sample = (f"random_dfa(n={n}, k={args.k}, seed={args.seed}, p={args.p}) {args.algo}PR, "
              f"{iters} passes; time = the reference's own RunStats.elapsed_ms")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.mean(ms), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (host-generated)",
            "config": config(args, world, iters, None),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_all}
    print(json.dumps(line), flush=True)


def make_family(args):
    from paper_2410_22764_b200 import generators as G
    if args.family == "chain":
        return G.chain_dfa(args.n)
    if args.family == "comb":
        return G.comb_dfa(args.n, 3)
    if args.family == "fib":
        return G.fib_dfa(args.n)
    if args.family == "bits":
        return G.bit_splitter(args.n)
    if args.family == "vlts":
        return G.vlts_dfa(args.vlts_m, args.n, args.k)
    raise ValueError(args.family)


def workload_name(args):
    if args.family == "random" and args.algo == "sort":
        tag = {(100_000_000, 4): " — north-star 1-GPU config (SURVEY 8(d) C5)",
               (100_000, 2): " — SURVEY 8(d) C1 (the reference's CPU-runnable config)"}
        return (f"sortPR on random_dfa(n={args.n:.0e}, k={args.k}, seed={args.seed}, p={args.p})"
                + tag.get((args.n, args.k), ""))
    fam = {"random": f"random_dfa(n={args.n}, k={args.k}, seed={args.seed})",
           "chain": f"chain_dfa({args.n})", "comb": f"comb({args.n},3)",
           "fib": f"fib_dfa({args.n})", "bits": f"bit_splitter({args.n})",
           "vlts": f"vlts(m={args.vlts_m}, n={args.n}, k={args.k})"}[args.family]
    return f"{args.algo} on {fam}"


def config(args, world, iters, blocks):
    return {"workload": workload_name(args), "family": args.family,
            "algo": args.algo, "n": args.n, "k": args.k, "passes": iters, "blocks": blocks,
            "sortpr_engine": args.sortpr_engine if args.algo == "sort" else None,
            "parallelism": "replicas" if world > 1 else "single",
            "l2": "inputs larger than L2 (delta = 4nk bytes)" if 4 * args.n * args.k > (126 << 20)
            else "L2 flushed between timed steps"}


# ----------------------------------------------------------------- our arm
def run_ours(args, rank: int, world: int, local: int):
    import numpy as np
    import torch
    import paper_2410_22764_b200 as dfm

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    eng = dfm.Engine(local)
    eng.set_sortpr_engine(args.sortpr_engine)
    stream = torch.cuda.current_stream(dev)
    eng.set_stream(stream.cuda_stream)
    algo = {"sort": dfm.Algo.sort, "naive": dfm.Algo.naive, "transpr": dfm.Algo.transpr,
            "naive_cas": dfm.Algo.naive_cas, "trans": dfm.Algo.trans}[args.algo]
    cfg = dfm.AlgoRunConfig(policy=dfm.RacePolicy.deterministic_min)
    seed = args.seed + rank
    if args.family == "random":
        dd = eng.random_dfa_device(args.n, args.k, seed, args.p)
    else:
        hd = make_family(args)
        args.n, args.k = hd.num_states, hd.alphabet_size
        dd = eng.upload(hd)
    flush = None
    if 4 * args.n * args.k <= (126 << 20):
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    for _ in range(args.warmup):
        nb, st = eng.run_device(algo, dd, cfg)
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # ---- timed region: device-resident input, CUDA events on the launch stream
    eng.profile_reset()
    eng.set_profiling(True)
    launches0 = eng.kernel_launches()
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize(dev)
    step_ms = []
    iters = None
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        nb, st = eng.run_device(algo, dd, cfg)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        iters = st.iterations
        assert st.status == dfm.RunStatus.ok
    torch.cuda.synchronize(dev)
    barrier()
    clk = clocks.stop()
    launches = eng.kernel_launches() - launches0
    eng.set_profiling(False)
    prof = eng.profile()
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    transitions = float(args.n) * args.k * iters * world
    value = transitions / (ms_per_step / 1e3)

    # ---- e2e: host DFA in pinned memory -> public API (H2D, run, D2H labels)
    e2e = None
    if not args.no_e2e:
        host = dd.download()
        pin_delta = torch.empty((args.k, args.n), dtype=torch.int32, pin_memory=True)
        pin_acc = torch.empty(args.n, dtype=torch.uint8, pin_memory=True)
        pin_delta.numpy()[:] = host.delta.view(np.int32)
        pin_acc.numpy()[:] = host.accepting
        hd = dfm.Dfa(args.n, args.k, pin_delta.numpy().view(np.uint32), pin_acc.numpy(), 0)
        del host
        out_pin = torch.empty(args.n, dtype=torch.int32, pin_memory=True)
        out_np = out_pin.numpy().view(np.uint32)
        run_host = {"sort": lambda: eng.sort_pr(hd, out=out_np),
                    "naive": lambda: eng.naive_pr(hd, dfm.PrOptions(
                        policy=dfm.RacePolicy.deterministic_min)),
                    "transpr": lambda: eng.trans_pr(hd, dfm.PrOptions(
                        policy=dfm.RacePolicy.deterministic_min)),
                    "naive_cas": lambda: eng.naive_pr_cas(hd),
                    "trans": lambda: eng.trans_minimize(hd)}[args.algo]
        run_host()  # warm the host path
        barrier()
        e_ms = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            r = run_host()
            e_ms.append((time.perf_counter() - t0) * 1e3)
            assert r.partition.num_blocks == nb
        et = torch.tensor([sum(e_ms) / len(e_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            torch.distributed.all_reduce(et, op=torch.distributed.ReduceOp.MAX)
        # when every block ends a singleton the canonical partition is the identity:
        # the library writes it on the host instead of reading 4n bytes back
        identity = args.algo == "sort" and nb == args.n
        e2e = {"value": transitions / (float(et.item()) / 1e3), "unit": UNIT,
               "ms_per_step": float(et.item()),
               "h2d_bytes_per_step": 4 * args.n * args.k + args.n,
               "d2h_bytes_per_step": 64 * (iters + 2) if identity else 4 * args.n,
               "how": "wall clock around Engine.sort_pr(host Dfa in pinned memory): H2D of "
                      "delta+accepting, all passes, per-pass device scalars read back, and "
                      "the canonical partition in the host buffer ("
                      + ("all singletons: identity labels written on the host" if identity
                         else "D2H of the labels") + ")"}
        del out_pin

    if rank != 0:
        return
    # ---- roofline of the dominant kernel family (measured live above)
    peak, peak_src = measured_peaks()
    fam = max(prof.items(), key=lambda kv: kv[1][1]) if prof else None
    roofline = None
    if fam is not None:
        name, (scopes, fms, fbytes) = fam
        achieved = (fbytes / 1e9) / (fms / 1e3) if fms > 0 else 0.0
        traffic = ncu_traffic(name, args)
        bound, unit = "hbm", "GB/s"
        if name == "gemm":  # tcgen05 kind::i8 squaring: the family counts 2*Vp^3 int8 ops
            bound, unit = "tensor", "TOP/s"
            achieved = (fbytes / 1e12) / (fms / 1e3) if fms > 0 else 0.0
            peak, peak_src = int8_peak()
        roofline = {"bound": bound, "kernel": name, "achieved": achieved, "peak": peak,
                    "unit": unit, "frac": achieved / peak, "traffic": traffic,
                    "peak_source": peak_src,
                    "share_of_step": fms / total_ms if total_ms > 0 else None,
                    "algorithmic_bytes_per_step": fbytes / args.steps,
                    "families_ms_per_step": {k: v[1] / args.steps for k, v in prof.items()}}
        # whole-iteration view with SURVEY 8(d)'s per-pass figure 8n(k+1)
        it_bytes = 8.0 * args.n * (args.k + 1) * iters
        roofline["iteration_view"] = {
            "algorithmic_bytes_per_step": it_bytes,
            "achieved": (it_bytes / 1e9) / (ms_per_step / 1e3),
            "frac": ((it_bytes / 1e9) / (ms_per_step / 1e3)) / peak}
    cpu = None
    if not args.no_cpu_baseline and world == 1 and args.algo == "sort" and args.family == "random":
        try:
            threads = os.cpu_count() or 1
            ns = min(args.n, args.cpu_sample_n)
            runs, citers, kind, cores, el = cpu_reference_sample(ns, args.k, args.seed, args.p,
                                                                 threads)
            cpu = {"value": runs[0], "unit": UNIT, "cores": cores, "kind": kind,
                   "sample": f"random_dfa(n={ns}, k={args.k}, seed={args.seed}, p={args.p}) "
                             f"sortPR, {citers} passes, {el:.0f} ms (reference RunStats)"}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": repr(exc)}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "wall_time_to_minimal_dfa_ms": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic: random_dfa generated on device, bit-exact with generators.hpp",
            "config": config(args, world, iters, nb), "e2e": e2e, "roofline": roofline,
            "cpu_baseline": cpu, "clocks": clk, "gpu_launches": launches,
            "step_ms": step_ms, "lib": dfm.lib_path()}
    print(json.dumps(line), flush=True)
    dd.free()


def run_sharded(args, rank: int, world: int, local: int):
    """N > 1: one random_dfa of n_total = n * N states, state-sharded over the ranks
    (paper_2410_22764_b200/sharded.py: NCCL all-gather of block ids + key exchange).
    Weak scaling: every GPU owns n states."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2410_22764_b200 as dfm
    from paper_2410_22764_b200.sharded import Comm, CudaShardOps, shard_bounds, sharded_sort_pr

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    eng = dfm.Engine(local)
    eng.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    ops = CudaShardOps(eng)
    comm = Comm()
    n_total = args.n * world
    lo, hi = shard_bounds(n_total, world, rank)
    delta, acc = ops.random_slice(n_total, args.k, args.seed, args.p, lo, hi - lo)
    for _ in range(args.warmup):
        r = sharded_sort_pr(delta, acc, n_total, lo, comm, ops)
    eng.profile_reset()
    eng.set_profiling(True)
    launches0 = eng.kernel_launches()
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    step_ms = []
    for _ in range(args.steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        r = sharded_sort_pr(delta, acc, n_total, lo, comm, ops)
        e1.record()
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = eng.kernel_launches() - launches0
    eng.set_profiling(False)
    prof = eng.profile()
    t = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t.item()) / args.steps
    transitions = float(n_total) * args.k * r.iterations
    value = transitions / (ms_per_step / 1e3)
    e2e = None
    if not args.no_e2e:
        # host slice in pinned memory -> H2D, sharded run, D2H of this rank's labels
        pin_d = torch.empty(delta.shape, dtype=torch.int32, pin_memory=True)
        pin_a = torch.empty(acc.shape, dtype=torch.uint8, pin_memory=True)
        pin_d.copy_(delta)
        pin_a.copy_(acc)
        out = torch.empty(hi - lo, dtype=torch.int32, pin_memory=True)
        e_ms = []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            rr = sharded_sort_pr(pin_d.to(dev, non_blocking=True), pin_a.to(dev, non_blocking=True),
                                 n_total, lo, comm, ops)
            out.copy_(rr.block_local)
            torch.cuda.synchronize(dev)
            e_ms.append((time.perf_counter() - t0) * 1e3)
        et = torch.tensor([sum(e_ms) / len(e_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": transitions / (float(et.item()) / 1e3), "unit": UNIT,
               "ms_per_step": float(et.item()),
               "h2d_bytes_per_step": (4 * args.k + 1) * n_total,
               "d2h_bytes_per_step": 4 * n_total,
               "how": "per rank: pinned host slice -> H2D, sharded sortPR, D2H of owned labels; "
                      "max over ranks"}
    if rank != 0:
        return
    peak, peak_src = measured_peaks()
    fam = max(prof.items(), key=lambda kv: kv[1][1]) if prof else None
    roofline = None
    if fam is not None:
        name, (scopes, fms, fbytes) = fam
        achieved = (fbytes / 1e9) / (fms / 1e3) if fms > 0 else 0.0
        roofline = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak,
                    "unit": "GB/s", "frac": achieved / peak, "traffic": None,
                    "peak_source": peak_src, "rank": 0,
                    "families_ms_per_step": {k: v[1] / args.steps for k, v in prof.items()}}
    cfg = config(args, world, r.iterations, r.num_blocks)
    cfg.update({"parallelism": f"state-sharded x{world} (NCCL all-gather + all-to-all)",
                "n_total": n_total, "workload": f"sharded sortPR on random_dfa(n={n_total:.2e}, "
                f"k={args.k}, seed={args.seed}) — {args.n:.0e} states per GPU (SURVEY 8(d) C5)",
                "hash_retries": r.retries})
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step,
            "wall_time_to_minimal_dfa_ms": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic: random_dfa slices generated on device, bit-exact with generators.hpp",
            "config": cfg, "e2e": e2e, "roofline": roofline, "cpu_baseline": None,
            "clocks": clk, "gpu_launches": launches, "step_ms": step_ms, "lib": dfm.lib_path()}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if (world > 1 or args.sharded) and args.algo == "sort" and not args.replicas:
            run_sharded(args, rank, world, local)
        else:
            run_ours(args, rank, world, local)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

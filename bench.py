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

Multi-GPU (N > 1): BASELINE configs[4] — ONE random_dfa(1e9, 4, seed 1)
state-sharded over the N ranks (strong scaling; NCCL all-gather of block ids +
key all-to-all per pass); timing is the max over ranks.  --replicas runs N
independent single-GPU minimizations instead (weak scaling).

Roofline: the headline is SURVEY 8(d)'s whole-iteration figure over the whole
step (8n(k+1) bytes per counted sortPR pass), with the executed passes beside
it; every kernel family's measured share of the step is listed.

cpu_baseline: the unmodified reference (oracle/_ref) on the same input at nproc
threads and at 1 thread (CPU model stated).

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified dfamin headers, input from its own generator) on the host cores, on
our arm's config; sortPR steps are one reference refinement pass each (see
run_reference_arm); rank 0 only.
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
    ap.add_argument("--c5-n", type=int, default=1_000_000_000,
                    help="N > 1 sortPR: states of the one random_dfa sharded over the N GPUs "
                         "(BASELINE configs[4], strong scaling)")
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


def measured_bf16():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except Exception:
        return None


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
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_generate(R, args):
    """The workload's input from the REFERENCE's own generators (generators.hpp) or the
    oracle's C generators for the builder-defined families — never libdfm."""
    from oracle import oracle as O
    if args.family == "random":
        return R.random_dfa(args.n, args.k, args.seed, args.p)
    if args.family == "chain":
        return R.chain_dfa(args.n)
    if args.family == "fib":
        return R.fib_dfa(args.n)
    if args.family == "bits":
        return R.bit_splitter(args.n)
    if args.family == "comb":
        return O.comb_dfa(args.n, 3)
    if args.family == "vlts":
        return O.vlts_dfa(args.vlts_m, args.n, args.k)
    raise ValueError(args.family)


def ref_run(R, algo, delta, acc, timeout_ms=3_600_000):
    """One run of the reference's own entry point for `algo`; RunStats timing.  On a
    timeout the reference still counts the passes it finished (core.hpp:190-199)."""
    if algo == "sort":
        return R.sort_pr(delta, acc, timeout_ms=timeout_ms)
    if algo == "naive":
        return R.naive_pr(delta, acc, "min", timeout_ms=timeout_ms)
    if algo == "naive_cas":
        return R.naive_pr(delta, acc, "min", fused_cas=True, timeout_ms=timeout_ms)
    if algo == "transpr":
        return R.trans_pr(delta, acc, "min", timeout_ms=timeout_ms, max_memory_bytes=64 << 30)
    if algo == "trans":
        return R.trans_minimize(delta, acc, timeout_ms=timeout_ms, max_memory_bytes=64 << 30)
    raise ValueError(algo)


def ref_bounded(R, args, delta, acc, budget_ms):
    """The reference on this input within a time budget: the whole run when it fits,
    else the passes it finished inside the budget (a bounded sample of the same
    workload); when not even one pass fits, a 10x smaller instance of the family."""
    n, k = acc.size, delta.shape[0]
    r = ref_run(R, args.algo, delta, acc, timeout_ms=int(budget_ms))
    if r.status == "ok":
        return (n * k * r.iterations / (r.call_ms / 1e3), r.call_ms, r.iterations,
                f"the whole run ({n} states, {r.iterations} passes)")
    if r.iterations > 0:
        return (n * k * r.iterations / (r.call_ms / 1e3), r.call_ms, r.iterations,
                f"the first {r.iterations} passes of the run ({n} states) inside a "
                f"{budget_ms / 1e3:.0f} s budget")
    if args.family in ("random", "vlts", "chain", "comb") and n >= 200_000:
        a1 = argparse.Namespace(**vars(args))
        a1.n = n // 10 if args.family != "vlts" else max(args.vlts_m, (n // 10) // args.vlts_m
                                                           * args.vlts_m)
        if args.family == "comb":
            a1.n = max(2, args.n // 10)
        d1, c1 = ref_generate(R, a1)
        v, ms, it, smp = ref_bounded(R, a1, d1, c1, budget_ms)
        return v, ms, it, f"{smp} of a smaller instance ({c1.size} states)"
    return None, r.call_ms, 0, "no pass finished inside the budget"


def cpu_baseline_for(args, delta, acc, our_iters, budget_ms=60_000):
    """cpu_baseline of our line: the unmodified reference (oracle/_ref) on the SAME input,
    at nproc threads and at 1 thread; rank 0, N = 1 only.  Each leg is
    bounded by `budget_ms` (ref_bounded)."""
    from oracle import oracle as O
    if not O.ref_available():
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                "sample": "oracle/_ref not built"}
    R = O.Reference()
    nproc = os.cpu_count() or 1
    out = {"unit": UNIT, "kind": "reference", "cpu_model": cpu_model(), "nproc": nproc}
    R.set_threads(nproc)
    v, ms, it, smp = ref_bounded(R, args, delta, acc, budget_ms)
    if "whole run" in smp and smp.startswith("the whole run ("):
        assert it == our_iters, (it, our_iters)
    out.update({"value": v, "cores": R.worker_count(), "ms": ms,
                "sample": f"reference {args.algo}, {R.worker_count()} threads: {smp}",
                "timing": "wall time of the reference call incl. its final canonicalize"})
    R.set_threads(1)
    if acc.size * delta.shape[0] > 100_000_000 and args.family in ("random", "vlts", "chain"):
        # one reference pass at 1 thread would take ~minutes here: a 10x smaller
        # instance of the same family (stated in the sample)
        a1 = argparse.Namespace(**vars(args))
        a1.n = (acc.size // 10 if args.family != "vlts"
                else max(args.vlts_m, acc.size // 10 // args.vlts_m * args.vlts_m))
        d1, c1 = ref_generate(R, a1)
        v1, ms1, it1, smp1 = ref_bounded(R, a1, d1, c1, budget_ms)
        smp1 = f"{smp1} of a 10x smaller instance of the family ({c1.size} states)"
        del d1, c1
    else:
        v1, ms1, it1, smp1 = ref_bounded(R, args, delta, acc, budget_ms)
    out["threads_1"] = {"value": v1, "ms": ms1, "passes": it1,
                        "sample": f"reference {args.algo}, 1 thread: {smp1}"}
    R.set_threads(0)
    if v1 is not None and (v is None or v1 > v):  # report the better as baseline
        out.update({"value": v1, "cores": 1, "ms": ms1, "sample": out["threads_1"]["sample"],
                    "nproc_run": {"value": v, "ms": ms, "sample": smp}})
    return out


def run_reference_arm(args, rank: int, world: int):
    """The reference's own CPU implementation (oracle/_ref, unmodified headers) on this
    box's host cores, on OUR arm's config/metric/unit.  Input from the reference's own
    generator.  sortPR steps are one refinement pass each (ref_sort_session_pass: the
    loop body of min_sort.hpp:100-118 over the reference's own functions; the fixpoint
    pass adds canonicalize) so K steps stay within minutes at 1e8 states; the timed
    steps start at pass 1, and when K is a multiple of the pass count they are exactly
    K/passes whole sort_pr runs.  Other algorithms: one whole reference run per step."""
    if rank != 0:
        return
    from oracle import oracle as O
    R = O.Reference()
    R.set_threads(os.cpu_count() or 1)
    t_all = time.perf_counter()
    line_extra = {}
    if args.algo == "sort" and args.family == "random":
        t0 = time.perf_counter()
        S = R.sort_session(args.n, args.k, args.seed, args.p)
        gen_s = time.perf_counter() - t0
        # above 2e8 states (C5, 1e9 at N > 1) a reference pass takes minutes: no warm-up
        # passes and the timed steps stop after one whole minimization
        huge = args.n > 200_000_000
        for _ in range(0 if huge else args.warmup):
            S.pass_()
        S.reset()
        ms, cycle, passes, blocks = [], [], None, None
        for _ in range(args.steps):
            if huge and passes is not None:
                break
            m, fresh, done = S.pass_()
            ms.append(m)
            cycle.append(m)
            if done:
                passes, blocks = (passes or len(cycle)), fresh
                line_extra.setdefault("ms_per_minimization", sum(cycle))
                cycle = []
        while passes is None:  # finish one cycle (untimed) to learn the pass count
            m, fresh, done = S.pass_()
            cycle.append(m)
            if done:
                passes, blocks = len(cycle), fresh
                line_extra.setdefault("ms_per_minimization", sum(cycle))
        S.close()
        value = len(ms) * float(args.n) * args.k / (sum(ms) / 1e3)
        line_extra["steps_timed"] = len(ms)
        step = "one sortPR refinement pass of the reference loop (the fixpoint pass adds " \
               "canonicalize); value = steps*n*k / sum of pass times"
        iters = passes
        sample = (f"reference sort_pr loop, {args.steps} passes over random_dfa(n={args.n}, "
                  f"k={args.k}, seed={args.seed}, p={args.p}) generated by the reference "
                  f"({gen_s:.0f} s, untimed); {passes} passes per minimization")
    else:
        delta, acc = ref_generate(R, args)
        args.n, args.k = acc.size, delta.shape[0]
        for _ in range(args.warmup):
            ref_run(R, args.algo, delta, acc)
        ms = []
        for _ in range(args.steps):
            r = ref_run(R, args.algo, delta, acc)
            ms.append(r.call_ms)
        iters, blocks = r.iterations, r.num_blocks
        value = args.steps * float(args.n) * args.k * iters / (sum(ms) / 1e3)
        step = ("one whole reference call, wall time incl. its final canonicalize "
                "(RunStats.elapsed_ms stops before it, min_sort.hpp:120-123)")
        sample = f"reference {args.algo} on the full workload, {iters} passes"
    cores = R.worker_count()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": statistics.mean(ms), "step": step, "higher_is_better": True,
            "scaling": scaling_of(args, world), "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (the reference's own generator)",
            "config": config(args, world, iters, blocks),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - t_all}
    line.update(line_extra)
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


def scaling_of(args, world):
    # N > 1 sortPR: one fixed random_dfa(1e9, 4) sharded over the N GPUs (configs[4])
    return "strong" if world > 1 and args.algo == "sort" and not args.replicas else "weak"


def config(args, world, iters, blocks):
    sharded = world > 1 and args.algo == "sort" and not args.replicas
    return {"workload": workload_name(args), "family": args.family,
            "algo": args.algo, "n": args.n, "k": args.k, "passes": iters, "blocks": blocks,
            "parallelism": (f"state-sharded x{world}" if sharded else
                            f"replicas x{world}" if world > 1 else "single"),
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

    # ---- e2e: host DFA -> public API (H2D, run, D2H labels), two host layouts:
    # pageable numpy rows (the reference's Dfa is std::vector rows: the drop-in case,
    # staged by the library through its pinned ring) and pinned rows
    e2e = None
    if not args.no_e2e:
        host = dd.download()
        pin_delta = torch.empty((args.k, args.n), dtype=torch.int32, pin_memory=True)
        pin_acc = torch.empty(args.n, dtype=torch.uint8, pin_memory=True)
        pin_delta.numpy()[:] = host.delta.view(np.int32)
        pin_acc.numpy()[:] = host.accepting
        hd_pin = dfm.Dfa(args.n, args.k, pin_delta.numpy().view(np.uint32), pin_acc.numpy(), 0)
        hd_page = dfm.Dfa(args.n, args.k, np.ascontiguousarray(host.delta),
                          np.ascontiguousarray(host.accepting), 0)
        del host
        out_pin = torch.empty(args.n, dtype=torch.int32, pin_memory=True)
        out_page = np.empty(args.n, np.uint32)

        def run_host(hd, out):
            pol = dfm.PrOptions(policy=dfm.RacePolicy.deterministic_min)
            return {"sort": lambda: eng.sort_pr(hd, out=out),
                    "naive": lambda: eng.naive_pr(hd, pol),
                    "transpr": lambda: eng.trans_pr(hd, pol),
                    "naive_cas": lambda: eng.naive_pr_cas(hd),
                    "trans": lambda: eng.trans_minimize(hd)}[args.algo]()

        def timed(hd, out):
            run_host(hd, out)  # warm the host path
            barrier()
            e_ms = []
            for _ in range(args.e2e_steps):
                t0 = time.perf_counter()
                r = run_host(hd, out)
                e_ms.append((time.perf_counter() - t0) * 1e3)
                assert r.partition.num_blocks == nb
            et = torch.tensor([sum(e_ms) / len(e_ms)], dtype=torch.float64, device=dev)
            if world > 1:
                torch.distributed.all_reduce(et, op=torch.distributed.ReduceOp.MAX)
            return float(et.item())

        ms_page = timed(hd_page, out_page)
        ms_pin = timed(hd_pin, out_pin.numpy().view(np.uint32))
        # when every block ends a singleton the canonical partition is the identity:
        # the library writes it on the host (a thread started at entry) instead of
        # reading 4n bytes back
        identity = args.algo == "sort" and nb == args.n and args.n >= (1 << 22)
        d2h = 64 * (iters + 2) if identity else 4 * args.n
        e2e = {"value": transitions / (ms_page / 1e3), "unit": UNIT, "ms_per_step": ms_page,
               "h2d_bytes_per_step": 4 * args.n * args.k + args.n, "d2h_bytes_per_step": d2h,
               "host_memory": "pageable (numpy rows, as the reference's std::vector Dfa)",
               "how": "wall clock around the public host-buffer call (Engine."
                      + {"sort": "sort_pr", "naive": "naive_pr", "transpr": "trans_pr",
                         "naive_cas": "naive_pr_cas", "trans": "trans_minimize"}[args.algo]
                      + "): H2D of delta+accepting (pageable rows staged by the library "
                        "through a pinned ring, several host threads), all passes, per-pass "
                        "scalars read back, the canonical partition in the host buffer ("
                      + ("all singletons: identity labels written on the host" if identity
                         else "D2H of the labels") + ")",
               "pinned": {"value": transitions / (ms_pin / 1e3), "ms_per_step": ms_pin,
                          "host_memory": "pinned (cudaMallocHost rows)"}}
        del out_pin, pin_delta, pin_acc, hd_pin, hd_page
        cpp = cpp_reference_types_e2e(args)
        if cpp is not None and "passes" in cpp:
            assert (cpp["passes"], cpp["blocks"]) == (iters, nb), cpp
            cpp["value"] = transitions / (cpp["ms_mean"] / 1e3)
        if cpp is not None:
            e2e["cpp_reference_types"] = cpp

    if rank != 0:
        dd.free()
        return
    peak, peak_src = measured_peaks()
    roofline = roofline_of(args, prof, ms_per_step, total_ms, iters, st.executed_passes,
                           peak, peak_src)
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        host = dd.download()
        try:
            cpu = cpu_baseline_for(args, host.delta, host.accepting, iters)
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": repr(exc)}
        del host
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "wall_time_to_minimal_dfa_ms": ms_per_step, "higher_is_better": True,
            "scaling": scaling_of(args, world), "vs_baseline": None, "dtype": "u32",
            "data": "synthetic: " + ("random_dfa generated on device, bit-exact with "
                                     "generators.hpp" if args.family == "random" else
                                     "host generator, uploaded once"),
            "config": config(args, world, iters, nb),
            "engine": args.sortpr_engine if args.algo == "sort" else "default",
            "passes_counted": iters, "passes_executed": st.executed_passes,
            "e2e": e2e, "roofline": roofline,
            "cpu_baseline": cpu, "clocks": clk, "gpu_launches": launches,
            "step_ms": step_ms, "lib": dfm.lib_path()}
    print(json.dumps(line), flush=True)
    dd.free()


def cpp_reference_types_e2e(args):
    """The C++ drop-in end to end (build/e2e_ref, tools/cpp/e2e_ref.cpp): the reference's
    own dfamin::Dfa (std::vector rows) from its generator, dfamin::b200::sort_pr, wall
    clock around the call.  None when the tool was not built or the workload has no
    generator there."""
    tool = os.path.join(ROOT, "build", "e2e_ref")
    if args.algo != "sort" or not os.path.exists(tool):
        return None
    if args.family == "random":
        cmd = [tool, "random", args.n, args.k, args.seed, 3]
    elif args.family == "vlts":
        cmd = [tool, "vlts", args.vlts_m, args.n, args.k, 3]
    else:
        return None
    try:
        r = subprocess.run([str(x) for x in cmd], capture_output=True, text=True, timeout=900)
        out = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as exc:  # pragma: no cover
        return {"error": repr(exc)}
    out["how"] = ("tools/cpp/e2e_ref.cpp: the reference's dfamin::Dfa from its own generator "
                  "(pageable std::vector rows), dfamin::b200::sort_pr (include/dfamin_b200.hpp "
                  "with DFAMIN_B200_USE_REFERENCE_TYPES), wall clock around the call incl. "
                  "upload, every pass and the canonical partition in the MinResult")
    return out


def roofline_of(args, prof, ms_per_step, total_ms, iters, executed, peak, peak_src):
    """Headline: SURVEY 8(d)'s whole-iteration figure over the whole step (every kernel):
    sortPR 8n(k+1) bytes per counted pass, naive/transPR n(16k'+8) per pass (upper
    bound), trans 2|V|^3 int8 ops per pass.  `families` lists every kernel family's
    measured time per step and share of the step (library profiler, CUDA events on the
    launch stream) with the dram bytes ncu measured for it (profiles/ncu_traffic.json,
    when this run is the workload captured there)."""
    n, k = float(args.n), args.k
    fams = {}
    for name, (scopes, fms, fbytes) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
        fams[name] = {"ms_per_step": fms / args.steps,
                      "share_of_step": fms / total_ms if total_ms > 0 else None,
                      "ncu_dram_bytes_per_step": ncu_traffic(name, args)}
    if args.algo == "trans":
        ops = 2.0 * (n * n) ** 3 * iters
        p8, p8src = int8_peak()
        achieved = ops / 1e12 / (ms_per_step / 1e3)
        out = {"bound": "tensor", "kernel": "whole minimization (every kernel of the step)",
               "achieved": achieved, "peak": p8, "unit": "TOP/s", "frac": achieved / p8,
               "traffic": None, "peak_source": p8src,
               "algorithmic": "2|V|^3 int8 ops per pass (|V| = n^2), SURVEY 8(d)",
               "families": fams}
        g = prof.get("gemm")
        if g and g[1] > 0:  # the tcgen05 kernels' EXECUTED int8 ops (live tile x K-block)
            ex = g[2] / 1e12 / (g[1] / 1e3)
            bf = 2.0 * measured_bf16()
            out["executed_ops_view"] = {
                "ops_per_step": g[2] / args.steps, "gemm_ms_per_step": g[1] / args.steps,
                "achieved": ex, "unit": "TOP/s", "frac_of_nominal_int8": ex / p8,
                "frac_of_2x_measured_bf16": ex / bf if bf else None,
                "note": "2*128*256*128 int8 ops per live (output tile, K block); all-zero "
                        "K blocks are skipped, so this is the tensor pipe's useful rate"}
        return out
    if args.algo == "sort":
        per_pass = 8.0 * n * (k + 1)
        formula = "8n(k+1) bytes per counted pass (SURVEY 8(d))"
    else:
        kk = k * (max(1, int(n).bit_length()) if args.algo == "transpr" else 1)
        per_pass = n * (16.0 * kk + 8)
        formula = "n(16k'+8) bytes per pass, k' = levels*k for transPR (SURVEY 8(d) upper bound)"
    it_bytes = per_pass * iters
    achieved = it_bytes / 1e9 / (ms_per_step / 1e3)
    traffic = ncu_traffic("step", args)
    out = {"bound": "hbm", "kernel": "whole minimization (every kernel of the step)",
           "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "traffic": traffic, "peak_source": peak_src, "algorithmic": formula,
           "algorithmic_bytes_per_step": it_bytes,
           "traffic_over_algorithmic": (traffic / it_bytes) if traffic else None,
           "families": fams}
    if args.algo == "sort" and executed and executed != iters:
        ex_bytes = per_pass * executed
        out["executed_passes_view"] = {
            "passes": executed, "algorithmic_bytes_per_step": ex_bytes,
            "achieved": ex_bytes / 1e9 / (ms_per_step / 1e3),
            "frac": ex_bytes / 1e9 / (ms_per_step / 1e3) / peak}
    return out


def run_sharded(args, rank: int, world: int, local: int):
    """N > 1 (or --sharded): ONE random_dfa(n = --c5-n, k, seed) state-sharded over the
    ranks through the C++ driver (libdfm dfm_sort_pr_sharded_dev; NCCL communicator
    owned by the library, bootstrapped over torch.distributed).  Strong scaling:
    the DFA is fixed, each rank owns ceil(n/N) states.  At N = 1 the protocol is
    forced (DFM_SHARD_PROTOCOL=1) so the line measures the sharded machinery itself;
    the single-GPU engine on the same input is timed beside it."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2410_22764_b200 as dfm
    from paper_2410_22764_b200.sharded import CudaShardOps, ShardedEngine

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world == 1:
        os.environ["DFM_SHARD_PROTOCOL"] = "1"
    se = ShardedEngine(local, rank, world, "nccl")
    eng = se.engine
    stream = torch.cuda.current_stream(dev)
    eng.set_stream(stream.cuda_stream)
    ops = CudaShardOps(eng)
    n_total = args.n
    lo, hi = se.bounds(n_total)
    delta, acc = ops.random_slice(n_total, args.k, args.seed, args.p, lo, hi - lo)
    out = torch.empty(max(hi - lo, 1), dtype=torch.int32, device=dev)
    for _ in range(args.warmup):
        nb, st = se.sort_pr_device(delta, acc, n_total, out)
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
        e0.record(stream)
        nb, st = se.sort_pr_device(delta, acc, n_total, out)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        assert st.status == dfm.RunStatus.ok
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
    iters = st.iterations
    transitions = float(n_total) * args.k * iters
    value = transitions / (ms_per_step / 1e3)
    e2e = None
    if not args.no_e2e:
        # pageable host slice -> the C-ABI host entry (dfm_sort_pr_sharded): H2D of the
        # owned rows, the sharded run, D2H of the owned labels; max over ranks
        host = dfm.Dfa(hi - lo, args.k, delta.cpu().numpy().view(np.uint32).copy(),
                       acc.cpu().numpy().copy(), 0)
        se.sort_pr(host, n_total)
        e_ms = []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            lab, nb2, st2 = se.sort_pr(host, n_total)
            e_ms.append((time.perf_counter() - t0) * 1e3)
            assert nb2 == nb
        et = torch.tensor([statistics.mean(e_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": transitions / (float(et.item()) / 1e3), "unit": UNIT,
               "ms_per_step": float(et.item()),
               "h2d_bytes_per_step": (4 * args.k + 1) * n_total, "d2h_bytes_per_step": 4 * n_total,
               "host_memory": "pageable",
               "how": "per rank: pageable host slice -> dfm_sort_pr_sharded (H2D of the owned "
                      "rows, the sharded run, D2H of the owned labels); max over ranks"}
    single = None
    if world == 1:
        # the single-GPU engine on the same DFA, generated on the device by
        # the same generator exactly as the default (single-engine) line does, after the
        # sharded context released its HBM (at 1e9 states both would not fit together)
        del delta, acc, out
        se.close()
        torch.cuda.empty_cache()
        e1 = dfm.Engine(local)
        e1.set_stream(stream.cuda_stream)
        dd = e1.random_dfa_device(n_total, args.k, args.seed, args.p)
        e1.run_device(dfm.Algo.sort, dd)
        sm = []
        for _ in range(max(1, min(args.steps, 5))):
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            nb1, st1 = e1.run_device(dfm.Algo.sort, dd)
            a1.record(stream)
            a1.synchronize()
            sm.append(a0.elapsed_time(a1))
        assert (nb1, st1.iterations) == (nb, iters)
        single = {"ms_per_step": statistics.mean(sm),
                  "sharded_over_single": ms_per_step / statistics.mean(sm)}
        dd.free()
        e1.close()
    if rank != 0:
        se.close()
        return
    peak, peak_src = measured_peaks()
    roofline = roofline_of(args, prof, ms_per_step, sum(step_ms), iters, st.executed_passes,
                           peak, peak_src)
    # NVLink: the per-pass exchange volume received by one rank (SURVEY 8(d) sharded row)
    roofline["nvlink"] = {
        "bytes_per_rank_per_step_upper": float(iters) * (4.0 * n_total * (world - 1) / world
                                                         + 16.0 * (n_total / world)
                                                         * (world - 1) / world),
        "peak_gbs_per_direction": 900.0,
        "note": "all-gather of ids (<= 4 B/state) + key/label exchange; measured on one GPU only"}
    cfg = config(args, world, iters, nb)
    cfg.update({"parallelism": f"state-sharded x{world} (C++ driver, NCCL all-gather + "
                               f"all-to-all)", "n_total": n_total,
                "workload": f"sharded sortPR on random_dfa(n={n_total:.0e}, k={args.k}, "
                            f"seed={args.seed}, p={args.p}) over {world} GPU(s) "
                            f"(BASELINE configs[4])"})
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step,
            "wall_time_to_minimal_dfa_ms": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic: random_dfa slices generated on device, bit-exact with "
                    "generators.hpp",
            "config": cfg, "passes_counted": iters, "passes_executed": st.executed_passes,
            "single_gpu_engine": single, "e2e": e2e, "roofline": roofline,
            "cpu_baseline": None, "clocks": clk, "gpu_launches": launches, "step_ms": step_ms,
            "lib": dfm.lib_path()}
    print(json.dumps(line), flush=True)
    se.close()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and args.algo == "sort" and not args.replicas:
        args.n = args.c5_n  # C5: one fixed DFA over all ranks
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

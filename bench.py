"""bench.py -- bounded subproblems/s of the B200 explorer on Taillard Ta021 (20x20),
frozen optimal UB 2297 (BASELINE.json configs[1]).

A step is one explorer round: select the pool (fill_buffer) at the target size,
expand + bound + prune + compact every child on the GPU (K2), push the survivors.
  value   device-resident explorer (pending tree in HBM), rounds timed with CUDA
          events inside the library; L2 flushed (256 MiB write) between rounds.
  e2e     same rounds through the reference-facing C-ABI with HOST buffers: host
          pending tree, parents H2D, K2, survivors D2H, host push; wall clock.
  --impl reference: the reference CPU explorer (oracle/_ref: the reference headers
          compiled in place; BackendSet over all host cores) on the same rounds.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--target T] [--impl ours|reference]
Multi-GPU (torchrun): each rank explores its own contiguous slice of the frontier
(split_slices, backend.hpp:73-84) and every round ends with the rank exchange of
paper_1206_4973_b200.parallel (incumbent + pending sizes all_gather, rebalancing
transfers every 4 rounds); per-GPU pool fixed (scaling "weak"); the value is all
ranks' bounded nodes over the max over ranks of (round device time + exchange).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

INSTANCES = {"ta021": (20, 20, 479340445, 2297), "ta022": (20, 20, 268827376, 2099),
             "ta051": (50, 20, 1539989115, 3847), "ta081": (100, 20, 450926852, 6202),
             "ta001": (20, 5, 873654221, 1279), "ta101": (200, 20, 2013025619, 11195)}
METRIC = "bounded subproblems/sec & explore time, Taillard 20x20/50x20, 1/2/4/8 B200"
INT32_LANES_PER_SM = 128  # ALU pipe 64 + FMA pipe 64 integer lanes / clk / SM (B300_MICROARCH)


def int_peak_gops(clock_mhz):
    """The integer roofline denominator, MEASURED on this pool's B200s by
    scripts/micro/intpeak.cu (profiles/r02_intpeak.json): the best 32-bit integer issue
    rate at full occupancy -- VIADDMNMX (ALU pipe) interleaved with IMAD (FMA pipe), 93.6
    lane-instructions/clk/SM, i.e. what the K1/K2 instruction mix can issue at most -- in
    Gop/s.  Falls back to the derived 148 x 128 lanes x clock when the file is missing."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_intpeak.json")) as f:
            d = json.load(f)
        mix = d["viaddmnmx+imad"]
        return mix["gops"], {
            "source": "measured: profiles/r02_intpeak.json (scripts/micro/intpeak.cu), "
                      "VIADDMNMX+IMAD at 2048 threads/SM",
            "lane_inst_per_clk_per_sm": mix["lane_inst_per_clk_per_sm"],
            "single_pipe_gops": d["viaddmnmx"]["gops"],
            "simd16x2_gops": d["viaddmnmx.s16x2"]["gops"],
            "derived_gops": 148 * INT32_LANES_PER_SM * clock_mhz * 1e6 / 1e9}
    except Exception:  # noqa: BLE001
        g = 148 * INT32_LANES_PER_SM * clock_mhz * 1e6 / 1e9
        return g, {"source": "derived: 148 SMs x 128 int32 lanes/clk x max SM clock"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--target", type=int, default=262144)
    ap.add_argument("--instance", default="ta021")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="explore", choices=["explore", "bound", "exhaust", "solve"],
                    help="explore: explorer rounds (configs 1-4); bound: K1 bound-only passes "
                         "over a synthetic pool in HBM (config 5, bounding stress); exhaust: "
                         "explore the whole tree (time-to-explore / proof of optimality); solve: "
                         "solve() from the identity-permutation UB (config 1 in the reference's "
                         "own mode), to optimality or --max-seconds")
    ap.add_argument("--ub", type=int, default=None,
                    help="--mode exhaust: frozen UB (default: the instance's UB + 1, so the "
                         "optimum is found and proven)")
    ap.add_argument("--max-seconds", type=float, default=1800.0,
                    help="--mode exhaust: wall-clock cap")
    ap.add_argument("--pool", type=int, default=8_000_000,
                    help="--mode bound: nodes in the synthetic pool (0: fill the GPU's free HBM)")
    ap.add_argument("--tuner", action="store_true",
                    help="adaptive pool size (autotune.hpp) instead of a fixed --target")
    ap.add_argument("--tuner-window", type=int, default=4)
    ap.add_argument("--group", type=int, default=0,
                    help="--mode exhaust, one process: explore with an fbb_group of this many "
                         "members (the in-library multi-device explorer; members on GPUs "
                         "0..G-1 when that many are visible, else all on GPU 0)")
    ap.add_argument("--exchange-every", type=int, default=4,
                    help="N > 1: explorer rounds per rank exchange (one library call each)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=60.0,
                    help="time cap of the reference arm's timed rounds")
    ap.add_argument("--cpu-sample", type=int, default=1_000_000,
                    help="bounded-node budget of the CPU baseline sample")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _clock_poll(device, stop, q, period):
    """Child process: NVML SM clock + throttle reasons every `period` s until `stop`."""
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(device)
    out = [pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)]
    while not stop.is_set():
        try:
            out.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        except Exception:  # noqa: BLE001
            pass
        time.sleep(period)
    q.put(out)


class ClockSampler:
    """SM clock and throttle reasons DURING the timed region, polled through NVML by a
    separate process (no GIL contention with the timed thread) every 10 ms -- each NVML
    query holds a driver lock for up to ~1 ms, so faster polling inflates the host side;
    the raw samples go to gpurun_out/clocks_<pid>.csv."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, device, period=0.01):
        import multiprocessing as mp

        try:
            import pynvml  # noqa: F401
        except Exception:  # noqa: BLE001
            self.proc = None
            return
        ctx = mp.get_context("spawn")
        self.stop, self.q = ctx.Event(), ctx.Queue()
        self.proc = ctx.Process(target=_clock_poll, args=(device, self.stop, self.q, period),
                                daemon=True)
        self.proc.start()
        time.sleep(0.5)  # NVML init in the child before the timed region starts

    def result(self):
        if self.proc is None:
            return None
        self.stop.set()
        try:
            out = self.q.get(timeout=30)
        except Exception:  # noqa: BLE001
            return None
        self.proc.join(timeout=10)
        max_mhz, samples = out[0], out[1:]
        if not samples:
            return None
        import pynvml

        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv"), "w") as f:
            for t, mhz, rs in samples:
                f.write(f"{t:.6f},{mhz},{rs:#x}\n")
        reasons = set()
        for _, _, rs in samples:
            for name, attr in self.REASONS.items():
                if rs & getattr(pynvml, attr, 0):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(m for _, m, _ in samples),
                "sm_max_mhz": max_mhz, "reasons": sorted(reasons),
                "samples": len(samples), "source": "NVML from a child process, ~10 ms polling"}


def k2_traffic(inst_name):
    """DRAM bytes (read + write) of one K2 launch from the committed ncu --set full capture
    (profiles/r02_k2_dram.json), when one exists for this instance; else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_k2_dram.json")) as f:
            d = json.load(f)[inst_name]
        return {"bytes_per_launch": d["dram_read_bytes"] + d["dram_write_bytes"],
                "children_per_launch": d["children_per_launch"], "kernel": d["kernel"],
                "source": "ncu --set full, profiles/r02_k2_dram.json"}
    except Exception:  # noqa: BLE001
        return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def explore_config(args, inst_name, world, tuner_desc=None):
    """The `config` of an explorer line -- identical in both arms (same workload)."""
    n, m, _, ub = INSTANCES[inst_name]
    return {"workload": f"{inst_name} {n}x{m} frozen UB {ub}, root pushed, prefill to a full pool, "
                        f"then rounds at pool target "
                        f"{'set by the adaptive tuner' if args.tuner else args.target}; step = one "
                        f"explorer round (select + expand/bound/prune + push)",
            "instance": inst_name,
            "pool_target": tuner_desc if (args.tuner and tuner_desc) else
                           ("adaptive" if args.tuner else args.target),
            "ub": ub, "parallelism": f"dp{world}",
            "l2": "flushed between timed rounds (256 MiB write)" if world == 1 else
                  f"flushed between timed exchange steps of {args.exchange_every} rounds "
                  f"(256 MiB write)"}


def reference_arm(args, inst_name):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import REF_SO, Oracle, Ref

    n, m, seed, ub = INSTANCES[inst_name]
    if args.mode == "bound":  # the reference evaluate_batch over random_node pools
        ref = Ref()
        cores = ref.detect_units()
        p = ref.generate_instance(n, m, seed)
        k, secs, _ = ref_evaluate_timed(ref, p, lambda k: ref.random_nodes(p, 0x5EED, k), cores,
                                        target_s=min(60.0, args.ref_seconds))
        value = k / secs
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "bounded subproblems/s", "n_gpus": world,
            "steps": 1, "warmup": 1, "ms_per_step": 1e3 * secs, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (Taillard generator; reference random_node pool)",
            "config": {"workload": f"{inst_name} {n}x{m} bounding stress: reference "
                                   f"BackendSet::evaluate over a random_node pool",
                       "instance": inst_name, "parallelism": "host threads"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "bounded subproblems/s", "cores": cores,
                             "kind": "reference", "sample": f"{k} random_node nodes, {secs:.1f} s"},
            "e2e": {"value": value, "unit": "bounded subproblems/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return
    cfg = explore_config(args, inst_name, world)
    if os.path.exists(REF_SO):
        ref = Ref()
        cores = ref.detect_units()
        p = ref.generate_instance(n, m, seed)
        # each step is one full reference round (~1 s at 262K children on 16 cores): the
        # timed steps stop after ~60 s so the arm ends within a few minutes at any K
        pre, rounds, secs = ref.bench_rounds(p, ub, args.target, args.warmup, args.steps,
                                             cores, max_seconds=args.ref_seconds)
        kind = "reference"
    else:  # the C restatement, single thread (reference not compiled on this host)
        orc = Oracle()
        p = orc.generate_instance(n, m, seed)
        t0 = time.perf_counter()
        res, rounds = orc.resolve(p, ub, [[]], targets=[args.target],
                                  budget=args.cpu_sample, max_trace=1 << 16)
        secs = [time.perf_counter() - t0]
        rounds = [tuple(r) for r in rounds]
        cores, kind, pre = 1, "port", 0
    bounded = sum(r[2] for r in rounds)
    total = sum(secs)
    value = bounded / total if total > 0 else 0.0
    line = {"metric": METRIC, "value": value, "unit": "bounded subproblems/s", "n_gpus": world,
            "steps": len(secs), "steps_requested": args.steps,
            "time_capped": len(secs) < args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / max(1, len(secs)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (Taillard generator, published seed)", "config": cfg,
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "bounded subproblems/s", "cores": cores,
                             "kind": kind,
                             "sample": f"{len(secs)} rounds after {pre} prefill + {args.warmup} "
                                       f"warm-up rounds, {bounded} bounded nodes; the reference "
                                       f"explorer (BackendSet over {cores} host threads)"},
            "e2e": {"value": value, "unit": "bounded subproblems/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "rounds": [list(r) for r in rounds]}
    print(json.dumps(line), flush=True)


def small_pool_batches(fbb, inst, ub, dev, targets=(4096, 16384, 32768), rounds=32, calls=10):
    """BASELINE configs[1]'s low end (the paper's 4 K-64 K pools) the way an explorer runs
    there: K rounds per fbb_explorer_run call on the HBM tree -- device-planned, so a batch of
    single-wave rounds is ONE cooperative launch of the persistent K2 (expand_v2.cu, BATCH).
    Per target: a fresh context from the root, prefill until a round reaches the target, 2
    warm-up calls, then `calls` timed calls of `rounds` rounds with the L2 flushed (256 MiB
    write) between calls.  device = bounded / the rounds' device-clock time; wall = bounded /
    wall clock of the calls (state upload, launch, download and sync included)."""
    import torch

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    out = {}
    for T in targets:
        ctx = fbb.Context(inst, dev)
        ctx.explorer_reset(fbb.NodeBatch.root(inst), ub, frozen=True)
        for _ in range(64):
            r = ctx.explorer_run([T], 1)
            if not r or r[0][2] >= T:
                break
        for _ in range(2):
            ctx.explorer_run([T], rounds)
        wall = devs = 0.0
        bounded = nr = launches = 0
        for c in range(calls):
            flush.fill_(c % 7)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            r, t = ctx.explorer_run([T], rounds, timing=True)
            wall += time.perf_counter() - w0
            devs += sum(x["round_ms"] for x in t) / 1e3
            bounded += sum(x[2] for x in r)
            nr += len(r)
            launches += sum(x["launches"] for x in t)
        ctx.close()
        out[str(T)] = {"rounds": nr, "bounded": bounded, "device_value": bounded / devs if devs else 0.0,
                       "wall_value": bounded / wall if wall else 0.0,
                       "us_per_round_device": 1e6 * devs / max(1, nr),
                       "us_per_round_wall": 1e6 * wall / max(1, nr), "gpu_launches": launches}
    return {"unit": "bounded subproblems/s", "rounds_per_call": rounds, "calls": calls,
            "l2": "flushed between calls (256 MiB write)", "targets": out}


def reference_api_e2e(target, steps):
    """The same workload driven through the calls a reference C++ user makes, with the
    reference's own PendingTree of heap Nodes on the host (tests/cpp/bench_dropin.cpp, built
    against the unmodified reference headers): gpu_round (K2 per round) and the reference
    resolve loop over GpuBackendSet (K1 per round).  None when the binary was not built."""
    import subprocess

    exe = os.path.join(ROOT, "tests", "cpp", "bin", "dropin_bench")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe, str(target), str(steps)], capture_output=True, text=True,
                             timeout=600)
        d = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)}
    d["unit"] = "bounded subproblems/s"
    d["timing"] = ("wall clock of the timed rounds, host Node packing/unpacking, PendingTree "
                   "pushes/pops and transfers included")
    return d


def cpu_baseline(inst_name, target, sample_nodes):
    """The reference CPU explorer (oracle/_ref) on bounded samples of the same workload: all
    host threads (BackendSet(k = nproc)) and one core (k = 1, the paper's Tcpu,
    PAPER.md:353-354).  The samples scale with the per-node cost (~n): ~2e6 / n nodes on
    one core, k/2 times that on k cores, rounds capped at the sample so that the first
    round never dominates (100x20 / 200x20 nodes cost ~1-4 ms each on one core)."""
    from oracle import REF_SO, Oracle, Ref

    n, m, seed, ub = INSTANCES[inst_name]
    if os.path.exists(REF_SO):
        ref = Ref()
        cores = ref.detect_units()
        p = ref.generate_instance(n, m, seed)
        one = max(2000, int(2e6 / n))
        many = min(sample_nodes, max(one, one * cores // 2))
        out = {}
        for k, budget in ((cores, many), (1, one)):
            tgt = min(target, budget)
            t0 = time.perf_counter()
            res, _, _ = ref.resolve(p, ub, [[]], targets=[tgt], budget=budget, backends=k,
                                    max_trace=1)
            secs = time.perf_counter() - t0
            out[k] = {"value": res["bounded"] / secs, "unit": "bounded subproblems/s", "cores": k,
                      "kind": "reference",
                      "sample": f"reference resolve from the root, pool target {tgt}, first "
                                f"{res['bounded']} bounded nodes ({res['rounds']} rounds, "
                                f"{secs:.1f} s, BackendSet({k}))"}
        line = dict(out[cores])
        line["single_core"] = out[1]
        return line
    orc = Oracle()
    p = orc.generate_instance(n, m, seed)
    t0 = time.perf_counter()
    res, _ = orc.resolve(p, ub, [[]], targets=[target], budget=sample_nodes // 20)
    secs = time.perf_counter() - t0
    return {"value": res["bounded"] / secs, "unit": "bounded subproblems/s", "cores": 1,
            "kind": "port", "sample": f"C restatement, resolve from the root, target {target}, "
                                      f"first {res['bounded']} bounded nodes ({secs:.1f} s)"}


def ref_evaluate_timed(ref, p, prefixes_of, cores, target_s=10.0):
    """Times the reference BackendSet::evaluate (all host cores) on a sample sized to take
    about target_s: a 64-node calibration call first.  prefixes_of(k) -> k prefixes."""
    t0 = time.perf_counter()
    ref.evaluate(p, prefixes_of(64), backends=cores)
    per = (time.perf_counter() - t0) / 64
    k = int(min(2_000_000, max(256, target_s / max(per, 1e-9))))
    pre = prefixes_of(k)
    t0 = time.perf_counter()
    lb, _ = ref.evaluate(p, pre, backends=cores)
    return k, time.perf_counter() - t0, lb


def bound_stress(args, inst_name):
    """BASELINE configs[4]: bound-only (K1 = CpuBackend::evaluate's drop-in) passes over a
    synthetic pool resident in HBM; a step = one pass over the whole pool.  The pool is
    random_node (tests/helpers.hpp:47-55) generated on the device (fbb_synth_pool);
    N GPUs each hold and bound their own pool (weak scaling, no collective)."""
    rank, world, local = dist_env()
    import torch

    dev = local if world > 1 and not os.environ.get("FBB_SAME_GPU") else 0
    torch.cuda.set_device(dev)
    backend = os.environ.get("FBB_DIST_BACKEND", "nccl")
    coll_dev = f"cuda:{dev}" if backend == "nccl" else "cpu"
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    import paper_1206_4973_b200 as fbb

    n, m, seed, ub = INSTANCES[inst_name]
    inst = fbb.generate_instance(n, m, seed)
    ctx = fbb.Context(inst, dev)
    cnt, W, P = args.pool, (n + 63) // 64, m * (m - 1) // 2
    cuda = f"cuda:{dev}"
    if cnt <= 0:  # --pool 0: the largest pool that fits this GPU's free HBM (4 GiB headroom)
        free_b, _ = torch.cuda.mem_get_info(dev)
        cnt = max(1 << 20, int((free_b - (4 << 30)) // (W * 8 + m * 4 + 4 + 4)))
        cnt -= cnt % 1024
    masks = torch.empty(cnt * W, dtype=torch.int64, device=cuda)
    heads = torch.empty(cnt * m, dtype=torch.int32, device=cuda)
    depth = torch.empty(cnt, dtype=torch.int32, device=cuda)
    lbs = torch.empty(cnt, dtype=torch.int32, device=cuda)
    ts = torch.cuda.Stream(device=cuda)  # K1 and the timing events on one (non-null) stream
    stream = ts.cuda_stream
    ctx.synth_pool(0x5EED + rank, cnt, 0, n - 1, masks.data_ptr(), heads.data_ptr(),
                   depth.data_ptr(), 0, stream)
    torch.cuda.synchronize()
    n_u = n - float(depth.sum(dtype=torch.int64).item()) / cnt  # no pool-sized temporaries

    def one_pass():
        ctx.bound_device(masks.data_ptr(), heads.data_ptr(), depth.data_ptr(), cnt, lbs.data_ptr(),
                         stream)

    for _ in range(args.warmup):
        one_pass()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev) if rank == 0 and not os.environ.get("FBB_NO_CLOCKS") else None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(ts)
    for _ in range(args.steps):
        one_pass()  # pool (cnt x ~100-300 B) > L2: every pass streams it from HBM
    ev1.record(ts)
    torch.cuda.synchronize()
    clocks = sampler.result() if sampler else None
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=coll_dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(t[0])
    total_nodes = cnt * args.steps * world

    e2e = None
    if not args.no_e2e:  # through fbb_bound: pinned host pool in, bounds out, every step
        sub = min(cnt, 1 << 22)
        hm = torch.empty(sub * W, dtype=torch.int64, pin_memory=True)
        hh = torch.empty(sub * m, dtype=torch.int32, pin_memory=True)
        hd = torch.empty(sub, dtype=torch.int32, pin_memory=True)
        hm.copy_(masks[: sub * W])
        hh.copy_(heads[: sub * m])
        hd.copy_(depth[:sub])
        hmn, hhn, hdn = hm.numpy().view(np.uint64), hh.numpy(), hd.numpy()
        out = torch.empty(sub, dtype=torch.int32, pin_memory=True).numpy()
        L = ctx.L
        for _ in range(2):
            ctx._check(L.fbb_bound(ctx.h, hmn, hhn, hdn, sub, out))
        steps_e = max(1, min(args.steps, 20))
        w0 = time.perf_counter()
        for _ in range(steps_e):
            ctx._check(L.fbb_bound(ctx.h, hmn, hhn, hdn, sub, out))
        es = time.perf_counter() - w0
        e2e = {"value": sub * steps_e * world / es, "unit": "bounded subproblems/s",
               "h2d_bytes_per_step": sub * (W * 8 + m * 4 + 4), "d2h_bytes_per_step": sub * 4,
               "timing": f"wall clock of fbb_bound over {sub} pinned host nodes per step "
                         f"(H2D + K1 + D2H), {steps_e} steps",
               "matches_device_pass": bool(np.array_equal(out, lbs[:sub].cpu().numpy()))}
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        from oracle import REF_SO, Ref

        if os.path.exists(REF_SO):
            ref = Ref()
            cores = ref.detect_units()
            def prefixes_of(k):  # the first k nodes of this pool, regenerated with prefixes
                pre = torch.empty(k * n, dtype=torch.uint8, device=cuda)
                dd = torch.empty(k, dtype=torch.int32, device=cuda)
                mm = torch.empty(k * W, dtype=torch.int64, device=cuda)
                hh2 = torch.empty(k * m, dtype=torch.int32, device=cuda)
                ctx.synth_pool(0x5EED, k, 0, n - 1, mm.data_ptr(), hh2.data_ptr(), dd.data_ptr(),
                               pre.data_ptr(), stream)
                torch.cuda.synchronize()
                dnp, pnp = dd.cpu().numpy(), pre.cpu().numpy().reshape(k, n)
                return [list(map(int, pnp[i, : dnp[i]])) for i in range(k)]

            ns, secs, ref_lb = ref_evaluate_timed(ref, inst.p, prefixes_of, cores)
            same = bool(np.array_equal(np.asarray(ref_lb, np.int32), lbs[:ns].cpu().numpy()))
            cpu = {"value": ns / secs, "unit": "bounded subproblems/s", "cores": cores,
                   "kind": "reference", "sample": f"first {ns} nodes of the pool through the "
                   f"reference BackendSet::evaluate ({secs:.1f} s, node construction included); "
                   f"bounds identical to K1: {same}"}
    ops_per_node = 4 * P * n_u + 2 * m * n_u  # SURVEY 8(a) W_K1
    peaks = measured_peaks()
    clock_mhz = (clocks or {}).get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0)
    int_peak, peak_src = int_peak_gops(clock_mhz)
    achieved = cnt * args.steps * ops_per_node / (ms / 1e3) / 1e9
    node_b = W * 8 + m * 4 + 4 + 4
    line = {
        "metric": METRIC, "value": total_nodes / (ms_max / 1e3), "unit": "bounded subproblems/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (Taillard generator, published seed; random_node pool generated on device)",
        "config": {"workload": f"{inst_name} {n}x{m} bounding stress: K1 (bound-only) passes over "
                               f"a synthetic pool of {cnt} nodes per GPU resident in HBM; step = "
                               f"one pass", "instance": inst_name, "pool_nodes": cnt,
                   "mean_unscheduled": n_u, "parallelism": f"dp{world} (own pool per GPU)",
                   "pool_gib": cnt * node_b / 2**30,
                   "l2": f"pool {cnt * node_b / 2**30:.2f} GiB > L2 (126 MB), no flush needed"},
        "e2e": e2e,
        "roofline": {"bound": "int32-alu", "kernel": ctx.kernels().split()[0][3:] + " (bound-only K1)",
                     "achieved": achieved, "peak": int_peak, "unit": "Gop/s",
                     "frac": achieved / int_peak, "traffic": None, "peak_source": peak_src,
                     "ops_per_node": ops_per_node,
                     "hbm": {"achieved": cnt * args.steps * node_b / (ms / 1e3) / 1e9,
                             "peak": peaks.get("hbm_gbs", 6553.9), "unit": "GB/s"}},
        "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": args.steps * world,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def exhaust(args, inst_name):
    """Time-to-explore: the frozen-UB exploration from the root run to exhaustion
    (resolve_workload, bench.hpp:63-114, with the pending tree in HBM).  With UB = opt + 1
    the run finds an optimal schedule's makespan and proves that nothing better exists
    (BASELINE configs[0]'s 'full B&B to optimality' for an instance whose tree fits).
    N > 1 (torchrun): each rank starts from its split_slices share of the first round's
    frontier and the ranks rebalance their pending trees (parallel.ParallelExplorer)
    until every rank is empty; the explore time is the max over ranks."""
    import torch

    rank, world, local = dist_env()
    dev = local if world > 1 and not os.environ.get("FBB_SAME_GPU") else 0
    torch.cuda.set_device(dev)
    backend = os.environ.get("FBB_DIST_BACKEND", "nccl")
    coll_dev = f"cuda:{dev}" if backend == "nccl" else "cpu"
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    import paper_1206_4973_b200 as fbb

    n, m, seed, ub0 = INSTANCES[inst_name]
    ub = args.ub if args.ub is not None else ub0 + 1
    inst = fbb.generate_instance(n, m, seed)
    ctx = fbb.Context(inst, dev)
    ctx.explorer_reset(fbb.NodeBatch.root(inst), ub, frozen=True)
    root_round = []
    if world > 1:  # the root round on every rank (deterministic), then split its frontier
        root_round = ctx.explorer_run([args.target], 1)
        frontier = ctx.explorer_pending()
        off, ln = fbb.split_slices(len(frontier), world)[rank]
        ctx.explorer_reset(fbb.nodes_from_prefixes(inst, frontier[off:off + ln]), ub, frozen=True)
    sampler = ClockSampler(dev) if rank == 0 and not os.environ.get("FBB_NO_CLOCKS") else None
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    dev_ms, rounds, transfers = 0.0, 0, 0
    group = None
    if world == 1 and args.group > 1:
        G = args.group
        devs = list(range(G)) if torch.cuda.device_count() >= G else [0] * G
        group = fbb.DeviceGroup(inst, devs)
        group.reset(fbb.NodeBatch.root(inst), ub, frozen=True)
        t0 = time.perf_counter()
        gs = group.run(args.target, max_steps=1 << 40, rounds_per_step=args.exchange_every,
                       balance_every=1)
        dev_ms, rounds, transfers = gs["device_ms_max"], gs["rounds"], gs["transfers"]
    elif world == 1:
        while True:
            r, t = ctx.explorer_run([args.target], 2000, timing=True)
            dev_ms += sum(x["round_ms"] for x in t)
            rounds += len(r)
            if ctx.explorer_state()["pending"] == 0 or time.perf_counter() - t0 > args.max_seconds:
                break
    else:
        from paper_1206_4973_b200.parallel import DevicePort, ParallelExplorer

        px = ParallelExplorer(DevicePort(ctx, frozen=True), n, device=coll_dev, balance_every=2,
                              exchange_every=args.exchange_every)
        while px.step(args.target):
            dev_ms += sum(x["round_ms"] for x in px.port.last_timings)
            if time.perf_counter() - t0 > args.max_seconds:
                break
        rounds, transfers = len(px.res.rounds), px.res.transfers
    wall = time.perf_counter() - t0
    clocks = sampler.result() if sampler else None
    st = ctx.explorer_state()
    if group is not None:  # totals over the group's members
        st = {"bounded": gs["bounded"], "branched": gs["branched"], "pruned": gs["pruned"],
              "leaves": gs["leaves"], "pending": gs["pending"], "found": bool(gs["found"]),
              "incumbent": gs["incumbent"]}
    best_mine = st["incumbent"] if st["found"] else 2**31 - 1
    tot = torch.tensor([st["bounded"], st["branched"], st["pruned"], st["leaves"], st["pending"]],
                       dtype=torch.int64, device=coll_dev)
    mx = torch.tensor([wall, dev_ms / 1e3], dtype=torch.float64, device=coll_dev)
    best = torch.tensor([best_mine], dtype=torch.int64, device=coll_dev)
    if world > 1:
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.SUM)
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(best, op=torch.distributed.ReduceOp.MIN)
    bounded, branched, pruned, leaves, pending = (int(x) for x in tot.cpu().tolist())
    bounded += sum(r[2] for r in root_round)
    wall_max, dev_max = (float(x) for x in mx.cpu().tolist())
    found = int(best.item()) < 2**31 - 1
    done = pending == 0
    if rank == 0:
        line = {
            "metric": METRIC, "value": bounded / wall_max, "unit": "bounded subproblems/s",
            "n_gpus": world, "steps": rounds, "warmup": 0,
            "ms_per_step": 1e3 * wall_max / max(1, rounds), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (Taillard generator, published seed; no dataset)",
            "config": {"workload": f"{inst_name} {n}x{m} exhaustive frozen-UB exploration from "
                                   f"the root at UB {ub}, pool target {args.target} per GPU",
                       "instance": inst_name, "ub": ub, "pool_target": args.target,
                       "parallelism": (f"fbb_group of {args.group} members in one process"
                                       if group is not None else
                                       f"dp{world}" + (" (pending-tree rebalancing)" if world > 1 else ""))},
            "explore_seconds": wall_max, "device_seconds": dev_max, "exhausted": done,
            "bounded": bounded, "branched": branched, "pruned": pruned, "leaves": leaves,
            "nodes_moved_between_gpus": transfers, "best_leaf": int(best.item()) if found else None,
            "group": ({"members": args.group, "devices": group.devices,
                       "exchange_ms": gs["exchange_ms"], "steps": gs["steps"],
                       "rounds_per_step": args.exchange_every} if group is not None else None),
            "proof": (f"optimum {int(best.item())}: no complete schedule below it exists"
                      if done and found else
                      f"no schedule below {ub}" if done else "time cap reached"),
            "clocks": clocks, "gpu_launches": rounds * 2,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def solve_mode(args, inst_name):
    """BASELINE configs[0] in the reference's own mode: solve() (search.hpp:124-174) from the
    identity-permutation makespan (search.hpp:131-137), strict-improvement incumbent with
    mid-batch updates, deepest-first LIFO selection at a fixed pool target, until the pending
    tree is empty (optimality proven) or --max-seconds.  Beside it, the reference's own
    solve() on the host cores (oracle/_ref, BackendSet over all threads) for a bounded node
    sample at the same pool target: its rate and the incumbent it reached."""
    import torch

    rank, world, local = dist_env()
    dev = local if world > 1 and not os.environ.get("FBB_SAME_GPU") else 0
    torch.cuda.set_device(dev)
    backend = os.environ.get("FBB_DIST_BACKEND", "nccl")
    coll_dev = f"cuda:{dev}" if backend == "nccl" else "cpu"
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    import paper_1206_4973_b200 as fbb

    n, m, seed, _ = INSTANCES[inst_name]
    inst = fbb.generate_instance(n, m, seed)
    ctx = fbb.Context(inst, dev)
    sampler = ClockSampler(dev) if rank == 0 and not os.environ.get("FBB_NO_CLOCKS") else None
    group, gs, px = None, None, None
    t0 = time.perf_counter()
    if world > 1:
        # one process per GPU (torchrun): rank 0 bounds the root, the other ranks start
        # empty with the same incumbent and are fed by rebalancing; every exchange step
        # min-allreduces the incumbent (the paper's UB allreduce)
        from paper_1206_4973_b200.parallel import DevicePort, ParallelExplorer

        if rank == 0:
            r0 = ctx.explorer_start_solve(None)
        else:
            ident = fbb.makespan(inst, list(range(n)))
            ctx.explorer_reset(fbb.NodeBatch.empty(inst), ident, frozen=False)
            r0 = (1, 0, 1, 1, 0, 0, ident, 1)
        px = ParallelExplorer(DevicePort(ctx, frozen=False), n, device=coll_dev, balance_every=1,
                              exchange_every=args.exchange_every)
        dev_ms, rounds, trace = 0.0, 1, []
        while px.step(args.target):
            dev_ms += sum(x["round_ms"] for x in px.port.last_timings)
            if time.perf_counter() - t0 > args.max_seconds:
                break
        res = px.finish()
        rounds += len(px.res.rounds)
        trace.append((round(time.perf_counter() - t0, 3), res.bounded, res.best))
    elif args.group > 1:
        # the in-library multi-device explorer: member 0 bounds the root, the others are fed
        # by rebalancing, and every step ends with the incumbent min-exchange (the paper's
        # UB allreduce)
        G = args.group
        devs = list(range(G)) if torch.cuda.device_count() >= G else [0] * G
        group = fbb.DeviceGroup(inst, devs)
        t0 = time.perf_counter()
        group.start_solve(None)
        r0 = (1, 0, 1, 1, 0, 0, fbb.makespan(inst, list(range(n))), 1)
        dev_ms, rounds, trace = 0.0, 1, []
        while True:
            gs = group.run(args.target, max_steps=100, rounds_per_step=args.exchange_every,
                           balance_every=1)
            dev_ms += gs["device_ms_max"]
            rounds += gs["rounds"]
            trace.append((round(time.perf_counter() - t0, 3), gs["bounded"], gs["incumbent"]))
            if gs["pending"] == 0 or time.perf_counter() - t0 > args.max_seconds:
                break
    else:
        r0 = ctx.explorer_start_solve(None)
        dev_ms, rounds, trace = 0.0, 1, []
        while True:
            r, t = ctx.explorer_run([args.target], 500, timing=True)
            dev_ms += sum(x["round_ms"] for x in t)
            rounds += len(r)
            st = ctx.explorer_state()
            trace.append((round(time.perf_counter() - t0, 3), st["bounded"], st["incumbent"]))
            if st["pending"] == 0 or not r or time.perf_counter() - t0 > args.max_seconds:
                break
    wall = time.perf_counter() - t0
    clocks = sampler.result() if sampler else None
    if px is not None:
        st0 = ctx.explorer_state()
        tot = torch.tensor([st0["bounded"], st0["branched"], st0["pruned"], st0["leaves"],
                            st0["pending"]], dtype=torch.int64, device=coll_dev)
        mx = torch.tensor([wall, dev_ms / 1e3], dtype=torch.float64, device=coll_dev)
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.SUM)
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        b, br, pr, lv, pe = (int(x) for x in tot.cpu().tolist())
        wall, dev_s = (float(x) for x in mx.cpu().tolist())
        dev_ms = 1e3 * dev_s
        st = {"pending": pe, "incumbent": px.res.best if px.res.best is not None else r0[6],
              "bounded": b, "branched": br, "pruned": pr, "leaves": lv}
        sched = px.res.schedule
        torch.distributed.destroy_process_group()
        if rank != 0:
            return
    elif group is not None:
        v, sched = group.best()
        st = {"pending": gs["pending"], "incumbent": v if v is not None else gs["incumbent"],
              "bounded": gs["bounded"], "branched": gs["branched"], "pruned": gs["pruned"],
              "leaves": gs["leaves"]}
    else:
        st = ctx.explorer_state()
        sched = st["schedule"]
    done = st["pending"] == 0
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        from oracle import REF_SO, Ref

        if os.path.exists(REF_SO):
            ref = Ref()
            cores = ref.detect_units()
            p = ref.generate_instance(n, m, seed)
            w0 = time.perf_counter()
            res, _, _ = ref.solve_trace(p, -1, targets=[args.target], budget=args.cpu_sample,
                                        backends=cores, max_trace=1)
            secs = time.perf_counter() - w0
            cpu = {"value": res["bounded"] / secs, "unit": "bounded subproblems/s", "cores": cores,
                   "kind": "reference",
                   "sample": f"reference solve() from the identity UB, pool target {args.target}, "
                             f"first {res['bounded']} bounded nodes in {secs:.1f} s; incumbent "
                             f"reached {res['optimum']}"}
    line = {
        "metric": METRIC, "value": st["bounded"] / wall, "unit": "bounded subproblems/s",
        "n_gpus": world, "steps": rounds, "warmup": 0, "ms_per_step": 1e3 * wall / max(1, rounds),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (Taillard generator, published seed; no dataset)",
        "config": {"workload": f"{inst_name} {n}x{m} solve() from the identity-permutation "
                               f"makespan, pool target {args.target}, to proven optimality "
                               f"(pending tree empty) or {args.max_seconds:.0f} s",
                   "instance": inst_name, "pool_target": args.target,
                   "parallelism": (f"fbb_group of {args.group} members (incumbent min-exchange "
                                   f"every {args.exchange_every} rounds)" if group is not None
                                   else f"dp{world}" + (f" (incumbent min-allreduce every "
                                                         f"{args.exchange_every} rounds)"
                                                         if world > 1 else ""))},
        "explore_seconds": wall, "device_seconds": dev_ms / 1e3, "exhausted": done,
        "optimum": st["incumbent"] if done else None, "incumbent": st["incumbent"],
        "schedule": sched, "schedule_makespan": fbb.makespan(inst, sched) if sched else None,
        "initial_ub": r0[6], "bounded": st["bounded"], "branched": st["branched"],
        "pruned": st["pruned"], "leaves": st["leaves"], "incumbent_trace": trace[:200],
        "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": rounds * 3,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.mode == "solve":
        solve_mode(args, args.instance)
        return
    if args.mode == "exhaust":
        exhaust(args, args.instance)
        return
    inst_name = args.instance
    if args.mode == "bound" and args.impl == "ours":
        bound_stress(args, inst_name)
        return
    if args.impl == "reference":
        reference_arm(args, inst_name)
        return
    rank, world, local = dist_env()
    import torch

    # FBB_SAME_GPU=1 + FBB_DIST_BACKEND=gloo: every rank on cuda:0, collectives over gloo
    # (exercises the N > 1 path on a one-GPU box; never used for reported numbers)
    dev = local if world > 1 and not os.environ.get("FBB_SAME_GPU") else 0
    torch.cuda.set_device(dev)
    backend = os.environ.get("FBB_DIST_BACKEND", "nccl")
    coll_dev = f"cuda:{dev}" if backend == "nccl" else "cpu"
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    import paper_1206_4973_b200 as fbb

    n, m, seed, ub = INSTANCES[inst_name]
    inst = fbb.generate_instance(n, m, seed)
    ctx = fbb.Context(inst, dev)
    T = args.target
    P = m * (m - 1) // 2

    # ---- prefill: rounds from the root until one reaches the pool target ------------------
    ctx.explorer_reset(fbb.NodeBatch.root(inst), ub, frozen=True)
    prefill = []
    while len(prefill) < 64:
        r = ctx.explorer_run([T], 1)
        if not r:
            break
        prefill.append(r[0])
        if r[0][2] >= T:
            break
    frontier = ctx.explorer_pending()
    px = None
    if world > 1:
        # each rank keeps its contiguous slice (split_slices, backend.hpp:73-84); from here on
        # every round ends with the rank exchange of parallel.ParallelExplorer (one all_gather
        # of [incumbent, pending, bounded] + rebalancing transfers every 4 rounds, NCCL)
        from paper_1206_4973_b200.parallel import DevicePort, ParallelExplorer

        off, ln = fbb.split_slices(len(frontier), world)[rank]
        frontier = frontier[off:off + ln]
        ctx.explorer_reset(fbb.nodes_from_prefixes(inst, frontier), ub, frozen=True)
    snapshot = fbb.nodes_from_prefixes(inst, frontier)

    def make_px():
        if world == 1:
            return None
        return ParallelExplorer(DevicePort(ctx, frozen=True), n, device=coll_dev,
                                balance_every=2, exchange_every=args.exchange_every)

    px = make_px()

    # --tuner: the pool target of every round comes from the adaptive tuner (autotune.hpp,
    # Algorithm 1 of the paper) with the B200 descriptor (grain = children per K2 chunk,
    # base_units = resident CTAs), observing each round's device time (search.hpp:155-165)
    tuner = fbb.Tuner(ctx.descriptor(), args.tuner_window) if args.tuner else None

    def one_round(timed, px):
        """One explorer round (+ the rank exchange when N > 1): (rounds, timings)."""
        tgt = tuner.target() if tuner else T
        if px is None:
            r, t = ctx.explorer_run([tgt], 1, timing=True)
        else:
            r, t = px_round(px, tgt)
        if tuner and r and t[0]["round_ms"] > 0:
            tuner.observe(r[0][2], t[0]["round_ms"] / 1e3)
        return r, t

    def px_round(px, tgt):
        """One exchange step: px.exchange_every rounds in one library call, then the rank
        exchange (charged to the step's last round)."""
        before = len(px.res.rounds)
        x0 = px.res.exchange_seconds
        px.step(tgt)
        r = px.res.rounds[before:]
        t = [dict(x) for x in px.port.last_timings] if r else []
        xm = 1e3 * (px.res.exchange_seconds - x0)
        if t:
            t[-1]["exchange_ms"] = xm
        else:
            t = [{"round_ms": 0.0, "k2_ms": 0.0, "launches": 0, "host_ms": 0.0, "sync_ms": 0.0,
                  "h2d_bytes": 0, "d2h_bytes": 0, "exchange_ms": xm}]
        return r, t

    # ---- device-resident explorer: W warm-up rounds, K timed rounds -------------------------
    for _ in range(args.warmup):
        one_round(False, px)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(dev) if rank == 0 and not os.environ.get("FBB_NO_CLOCKS") else None
    rounds, timing, wall, flush_s = [], [], 0.0, 0.0
    for _ in range(args.steps):
        if len(rounds) >= args.steps:  # N > 1: a step of px runs exchange_every rounds
            break
        f0 = time.perf_counter()
        flush.fill_(rank + len(rounds) % 7)  # L2 flush (> 126 MB) between timed rounds
        torch.cuda.synchronize()
        w0 = time.perf_counter()  # wall clock of the round itself (the flush excluded)
        flush_s += w0 - f0
        r, t = one_round(True, px)
        wall += time.perf_counter() - w0
        if px is None and not r:
            break
        if px is not None and px.res.exhausted:
            timing += t
            break
        rounds += r
        timing += t
    torch.cuda.synchronize()
    clocks = sampler.result() if sampler else None
    # device time per rank: the rounds' CUDA-event time plus the rank exchange (N > 1)
    dev_ms = sum(t["round_ms"] + t.get("exchange_ms", 0.0) for t in timing)
    k2_ms = sum(t["k2_ms"] for t in timing)
    bounded = sum(r[2] for r in rounds)
    branched = sum(r[1] for r in rounds)
    leaves = sum(r[5] for r in rounds)
    survivors = sum(r[3] for r in rounds)
    launches = sum(t["launches"] for t in timing)
    stats = torch.tensor([dev_ms, k2_ms, wall, bounded, branched, leaves, survivors, launches,
                          len(rounds)], dtype=torch.float64, device=coll_dev)
    if world > 1:
        import torch.distributed as dist

        mx = stats.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        dev_ms_max, wall_max = float(mx[0]), float(mx[2])
        bounded_all, launches_all = float(sm[3]), float(sm[7])
    else:
        dev_ms_max, wall_max, bounded_all, launches_all = dev_ms, wall, bounded, launches

    # ---- e2e: same rounds with the pending tree in pinned HOST memory, through the C-ABI:
    # every round uploads its parents and writes only the survivors back into host memory
    e2e = None
    if not args.no_e2e:
        ctx.explorer_set_residency(True)
        ctx.explorer_reset(snapshot, ub, frozen=True)
        pxe = make_px()
        if pxe is None and tuner is None and args.warmup >= 2:
            ctx.explorer_run([T], args.warmup)  # as one call: the batch's graph is built here
        else:
            for _ in range(args.warmup):
                one_round(False, pxe)
        if world > 1:
            torch.distributed.barrier()
        e_rounds, e_tim, e_secs = [], [], 0.0
        if pxe is None and tuner is None:
            # one C-ABI call runs the K rounds (device-planned batches of up to 64 rounds, no
            # host round trip between them); the host tree is read and written over the
            # link every round
            w0 = time.perf_counter()
            e_rounds, e_tim = ctx.explorer_run([T], args.steps, timing=True)
            e_secs = time.perf_counter() - w0
        else:
            for _ in range(args.steps):
                if len(e_rounds) >= args.steps:
                    break
                w0 = time.perf_counter()
                r, t = one_round(True, pxe)
                e_secs += time.perf_counter() - w0
                if (pxe is None and not r) or (pxe is not None and pxe.res.exhausted):
                    break
                e_rounds += r
                e_tim += t
        ctx.explorer_set_residency(False)
        stepsd = max(1, len(e_rounds))
        e_stats = torch.tensor([e_secs, sum(r[2] for r in e_rounds)], dtype=torch.float64,
                               device=coll_dev)
        if world > 1:
            mx = e_stats.clone()
            torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
            sm = e_stats.clone()
            torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM)
            e_secs_max, e_bounded = float(mx[0]), float(sm[1])
        else:
            e_secs_max, e_bounded = e_secs, float(e_stats[1])
        e2e = {"value": e_bounded / e_secs_max if e_secs_max > 0 else 0.0,
               "unit": "bounded subproblems/s",
               "h2d_bytes_per_step": sum(t["h2d_bytes"] for t in e_tim) // stepsd,
               "d2h_bytes_per_step": sum(t["d2h_bytes"] for t in e_tim) // stepsd,
               "rounds_match_device_explorer": [tuple(r) for r in e_rounds] == [
                   tuple(r) for r in rounds[: len(e_rounds)]],
               "per_round_ms": {"wall": 1e3 * e_secs / stepsd,
                                "device": sum(t["round_ms"] for t in e_tim) / stepsd,
                                "k2": sum(t["k2_ms"] for t in e_tim) / stepsd,
                                "library_host": sum(t["host_ms"] for t in e_tim) / stepsd,
                                "sync_wait": sum(t["sync_ms"] for t in e_tim) / stepsd},
               "timing": "wall clock of fbb_explorer_run over the K rounds with the pending tree in "
                         "pinned, device-mapped host memory (parents read and survivors written "
                         "over the host link every round)"}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6528.7)
    clock_mhz = (clocks or {}).get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0)
    int_peak, peak_src = int_peak_gops(clock_mhz)  # Gop/s
    internal = bounded - leaves
    # algorithmic int32 ops: per parent scan P*n, per child P*15 + 6m
    ops = P * (n * max(0, branched - leaves // 2) + 15 * internal) + 6 * m * bounded
    node_b = ((n + 63) // 64) * 8 + m * 4 + n
    alg_bytes = (branched * node_b) + survivors * (2 * node_b + 4)  # parents in, survivors staged+pushed
    k2_s = k2_ms / 1e3
    roofline = {
        "bound": "int32-alu",
        "kernel": ctx.kernels().split()[1][3:] + " (fused expand+bound+prune+compact)",
        "achieved": ops / k2_s / 1e9 if k2_s > 0 else 0.0, "peak": int_peak, "unit": "Gop/s",
        "frac": (ops / k2_s / 1e9) / int_peak if k2_s > 0 else 0.0,
        "traffic": (k2_traffic(inst_name) or {}).get("bytes_per_launch"),
        "traffic_source": k2_traffic(inst_name),
        "ops_per_child": ops / max(1, bounded),
        "peak_source": peak_src,
        "hbm": {"achieved": alg_bytes / k2_s / 1e9 if k2_s > 0 else 0.0, "peak": hbm_peak,
                "unit": "GB/s", "frac": (alg_bytes / k2_s / 1e9) / hbm_peak if k2_s > 0 else 0.0},
        "k2_share_of_round": k2_ms / dev_ms if dev_ms > 0 else 0.0,
        "k2_time_source": ("CUDA events around K2 (FBB_PDL=0)" if os.environ.get("FBB_PDL") == "0" else
                           "device clock (%globaltimer) stamps in the round state: first K2 CTA start .. "
                           "last K2 CTA end (place_kernel is K2's programmatic dependent launch, so no "
                           "event can sit between them); rounds themselves are CUDA-event timed"),
    }
    ref_api = None
    small = None
    if not args.no_e2e and world == 1 and inst_name == "ta021" and not args.tuner:
        ref_api = reference_api_e2e(T, min(args.steps, 20))
        small = small_pool_batches(fbb, inst, ub, dev)
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cpu = cpu_baseline(inst_name, T, args.cpu_sample)
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)}
    steps_done = len(rounds)
    line = {
        "metric": METRIC,
        "value": bounded_all / (dev_ms_max / 1e3) if dev_ms_max > 0 else 0.0,
        "unit": "bounded subproblems/s",
        "n_gpus": world, "steps": steps_done, "warmup": args.warmup,
        "ms_per_step": dev_ms_max / max(1, steps_done),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (Taillard generator, published seed; no dataset)",
        "config": explore_config(args, inst_name, world),
        "tuner": ({"best_batch": tuner.best_batch(), "phase": tuner.phase().name,
                   "targets": [r[0] for r in rounds]} if tuner else None),
        "kernels": ctx.kernels(),
        "wall_value": bounded_all / wall_max if wall_max > 0 else 0.0,
        "wall_breakdown_ms_per_step": {
            "round_wall": 1e3 * wall / max(1, len(rounds)),
            "library_host": sum(t["host_ms"] for t in timing) / max(1, len(timing)),
            "library_sync_wait": sum(t["sync_ms"] for t in timing) / max(1, len(timing)),
            "device_events": dev_ms / max(1, len(timing)),
            "l2_flush_untimed": 1e3 * flush_s / max(1, len(rounds))},
        "e2e": e2e, "e2e_reference_api": ref_api, "small_pool_batches": small, "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "gpu_launches": int(launches_all),
        "rounds": [list(r) for r in rounds],
        "prefill_rounds": len(prefill),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

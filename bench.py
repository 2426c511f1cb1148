#!/usr/bin/env python
"""bench.py — PSTF field cache (keygen + insert + blend + lookup) on B200.

Workload (BASELINE.json configs[1]): a 1920x1080 1 spp x 4-bounce
synthetic Cornell vertex stream (8,294,400 vertices/iteration, 276 B/vertex canonical fp64 SoA
record), spatio-directional keys, three field stores (Lo, Lo\\E, FLi) of 2^22 slots each,
base cell = diameter/256.  One step = one progressive iteration: the fused onVertex pass
(lookups on committed state + key generation + counter/accumulate updates incl. deterministic
placement of new keys) followed by endFrame on the three stores (blend + cap + eviction).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

`value` is device-timed with CUDA events (inputs resident in HBM, 8 distinct iteration streams
of 2.29 GB each cycled, i.e. inputs larger than L2); `e2e` is the same metric through the C ABI
with pinned HOST vertex arrays copied in every step; `roofline` covers the dominant kernel
(k_vertex_pass) and `step_roofline` the whole iteration against SURVEY.md §8d's algorithmic
bytes (276 B/vertex + 172 B/touched cell).  `--impl reference` times the reference's own
FieldStore (oracle/_ref, compiled from /root/reference) driven by the onVertex replay on all
host cores.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "filtered path vertices/sec (insert+blend+lookup) 1080p×4 bounces; % HBM roofline"
UNIT = "vertices/s"
BYTES_PER_VERTEX = 276
BYTES_PER_TOUCHED = 172
DATA = "synthetic (pstf_synth.h Cornell-box generator, IEEE-exact, seed 0x5EED)"
DIAMETER = math.sqrt(12.0)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None,
                   help="timed iterations (default 20; config 5: 128, BASELINE configs[4])")
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--bounces", type=int, default=4)
    p.add_argument("--capacity-log2", type=int, default=None,
                   help="slots per store (default 2^22; config 4: 2^24; config 5: the next power "
                        "of two >= 2 x L2 / slot bytes, SURVEY.md 8(d))")
    p.add_argument("--streams", type=int, default=8)
    p.add_argument("--mode", default="atomic", choices=["atomic", "ordered"])
    p.add_argument("--e2e-steps", type=int, default=4)
    p.add_argument("--cpu-seconds", type=float, default=20.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--force-sharded", action="store_true",
                   help="testing: run the multi-GPU iteration (NCCL) even at world 1")
    p.add_argument("--scaling", default=None, choices=["weak", "strong"],
                   help="N>1: weak = every rank traces its own 1 spp of the frame (default for "
                        "configs 2/3/5); strong = the ranks split one frame into image stripes "
                        "(default for config 4)")
    p.add_argument("--config", type=int, default=2, choices=[2, 3, 4, 5],
                   help="BASELINE.json config: 2 = 1080p x4 (default, the metric's workload); "
                        "3 = + CV lookup at every vertex; 4 = 4K x6 at 2^24 slots; 5 = drifting "
                        "camera (+0.02/iter), 2^20 slots so eviction engages")
    a = p.parse_args()
    if a.scaling is None:
        a.scaling = "strong" if a.config == 4 else "weak"
    if a.steps is None:
        a.steps = 128 if a.config == 5 else 20
    if a.config == 4:
        a.width, a.height, a.bounces, a.streams = 3840, 2160, 6, 2
    if a.capacity_log2 is None:
        a.capacity_log2 = {4: 24, 5: config5_capacity_log2()}.get(a.config, 22)
    return a


SLOT_BYTES = 8 + 32 + 32 + 24 + 8 + 4  # meta, com, acc, key fields, placement holds, list


def config5_capacity_log2():
    """the next power of two >= 2 x L2 / slot bytes (L2 read from the
    device, cudaDevAttrL2CacheSize; 126.5 MB on B200 -> 2^22)"""
    l2 = 126 * 1024 * 1024
    try:
        import torch
        if torch.cuda.is_available():
            l2 = torch.cuda.get_device_properties(0).L2_cache_size
    except Exception:
        pass
    need = 2 * l2 // SLOT_BYTES
    return max(10, int(need - 1).bit_length())


WORKLOADS = {
    2: "config2: 1920x1080 1spp x4 bounces synthetic Cornell vertex stream, spatio-directional "
       "keys, Lo/LoE/FLi stores x 2^22 slots, base=diam/256",
    3: "config3: config 2 with the glossy materials of staircase_glossy.scene (Phong albedo 0.6, "
       "exponent 48 on floor and back wall) + CV lookup (Lo\\E query) at every vertex",
    4: "config4: 3840x2160 1spp x6 bounces, Lo/LoE/FLi x 2^24 slots",
    5: "config5: config 2 with the camera drifting +0.02/iteration, 128 iterations, stores at "
       "2 x L2 (next power of two), inputs regenerated untimed",
}


def bench_config(args, streams, world, multi=None):
    """the `config` object both arms print (identical for the same command line); multi: the
    multi-GPU protocol runs (default: world > 1; --force-sharded runs it on one rank)"""
    multi = world > 1 if multi is None else multi
    W, H, B = args.width, args.height, args.bounces
    return {
        "workload": WORKLOADS[args.config], "vertices_per_iter": W * H * B,
        "capacity_log2": args.capacity_log2, "stores": 3, "mode": args.mode,
        "iteration_streams": streams,
        "inputs": "%d distinct iteration streams of %.2f GB cycled (inputs larger than L2)"
                  % (streams, BYTES_PER_VERTEX * W * H * B / 1e9),
        "parallelism": "single GPU" if not multi else
                       (f"{world} ranks, each tracing its own 1 spp of the frame (weak scaling)"
                        if args.scaling == "weak" else
                        f"{world} ranks, one frame split into {world} image stripes (strong "
                        "scaling)") + ", one field cache: replicated stores, live-slot "
                        "accumulators all-reduced over "
                        + ("NCCL" if os.environ.get("PSTF_BENCH_BACKEND", "nccl") == "nccl"
                           else os.environ["PSTF_BENCH_BACKEND"] + " (bench.py test mode)"),
    }


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML every ~2 ms; the
    nvidia-smi CLI as a fallback)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self._stop.is_set():
                    try:
                        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
                        self.samples.append((mhz, rs, util))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.t:
            self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = sorted(x[0] for x in self.samples)
        reasons = sorted({name for x in self.samples for bit, name in self.REASONS.items()
                          if x[1] & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------- CPU reference leg
def cpu_reference_run(args, steps, warmup, budget_s, streams=2):
    """The reference FieldStore (oracle/_ref) + onVertex replay, non-deterministic mode on all host
    threads (EstimatorRun::renderFrame threading, estimators.cpp:566-608).  Each step replays a
    path sample (all bounces of a random subset of the frame's paths) and runs endFrame on the
    three stores; the sample is sized so warmup+steps fit the time budget."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po
    kind = "reference" if po.ref_available() else "port"
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    base = DIAMETER / 256.0
    W, H, B = args.width, args.height, args.bounces
    n_paths = W * H
    n_full = n_paths * B
    gen_threads = max(1, threads)
    def sample(buf, frac, seed):
        k = max(1, int(n_paths * frac))
        rng = np.random.default_rng(seed)
        paths = np.sort(rng.choice(n_paths, size=k, replace=False))
        idx = (np.arange(B)[:, None] * n_paths + paths[None, :]).reshape(-1)
        f64, flags = po.soa_views(buf, n_full)
        m = len(idx)
        out = np.zeros(34 * m + (m + 1) // 2, np.float64)
        out[:34 * m] = f64[:, idx].reshape(-1)
        out[34 * m:].view(np.uint32)[:m] = flags[idx]
        return out, m

    if kind == "reference":
        mk = lambda k: po.RefStore(po.Config.make(kind=k, capacity_log2=args.capacity_log2,
                                                  base_cell_size=base))
    else:
        mk = lambda k: po.OracleStore(po.Config.make(kind=k, capacity_log2=args.capacity_log2,
                                                     base_cell_size=base))
    stores = [mk(k) for k in (po.KIND_LO, po.KIND_LOE, po.KIND_FLI)] + [None]

    def step(sbuf, m):
        t0 = time.perf_counter()
        if kind == "reference":
            po.vertex_pass_ref(*stores, sbuf, m, deterministic=False, threads=threads,
                               chunk=W)
        else:
            po.vertex_pass_oracle(*stores, sbuf, m, deterministic=False)
        t1 = time.perf_counter()
        for s in stores[:3]:
            s.end_frame()
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1

    # calibrate on a small sample, then size the sample to the budget; the iteration streams
    # are generated one at a time and only their samples kept (the GPU arm cycles the same
    # `streams` iteration streams)
    scene = 1 if args.config == 3 else 0
    buf0 = po.synth_generate(W, H, B, iteration=0, threads=gen_threads, scene=scene)[0]
    cal, cm = sample(buf0, 1.0 / 64, 1)
    tp, te = step(cal, cm)
    rate = cm / max(tp, 1e-9)
    per_step = budget_s / max(1, steps + warmup)
    frac = max(1.0 / 64, min(1.0, (per_step - te) * rate / n_full)) if per_step > te else 1.0 / 64
    samples = [sample(buf0, frac, 100)]
    del buf0
    for i in range(1, streams):
        bi = po.synth_generate(W, H, B, iteration=i, threads=gen_threads, scene=scene)[0]
        samples.append(sample(bi, frac, 100 + i))
        del bi
    for i in range(warmup):
        step(*samples[i % len(samples)])
    tot_v, tot_t, t_pass, t_ef = 0, 0.0, 0.0, 0.0
    for i in range(steps):
        sbuf, m = samples[(warmup + i) % len(samples)]
        a, b = step(sbuf, m)
        tot_v += m
        tot_t += a + b
        t_pass += a
        t_ef += b
    value = tot_v / tot_t
    phases = None
    if kind == "reference":  # keygen / lookup / insert / endFrame separately
        sbuf, m = samples[0]
        ph = po.vertex_pass_phases_ref(*stores[:3], sbuf, m, threads)
        scale = n_full / m
        phases = {k: round(v * scale, 2) for k, v in ph.items()}
        phases["endFrame"] = round(t_ef / steps * 1e3, 2)
    return {
        "value": value, "unit": UNIT, "cores": threads if kind == "reference" else 1,
        "kind": kind, "host": po.host_info(),
        "phases_ms_per_iteration": phases,
        "sample": (f"{frac:.4f} of the {n_full}-vertex iteration per step, {len(samples)} "
                   f"iteration streams cycled "
                   f"({samples[0][1]} vertices = all {B} bounces of a random path subset), "
                   f"{steps} steps after {warmup} warm-up; each step = onVertex replay "
                   f"({'non-deterministic, ' + str(threads) + ' std::threads' if kind == 'reference' else '1 thread'}) "
                   f"+ endFrame x3 at 2^{args.capacity_log2}; pass {t_pass / steps * 1e3:.1f} ms, "
                   f"endFrame {t_ef / steps * 1e3:.1f} ms per step; full-iteration extrapolation "
                   f"{n_full / (t_pass / steps * n_full / samples[0][1] + t_ef / steps):.4g} v/s"),
        "ms_per_step": tot_t / steps * 1e3,
    }


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0  # under a launcher rank 0 alone times the host path
    r = cpu_reference_run(args, args.steps, args.warmup, budget_s=150.0,
                          streams=max(1, args.streams))
    line = {
        "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64", "data": DATA, "impl": "reference", "launched_ranks": world,
        "config": bench_config(args, max(1, args.streams), args.gpus),
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                         "sample": r["sample"], "host": r["host"],
                         "phases_ms_per_iteration": r["phases_ms_per_iteration"]},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- B200 leg
def run_b200(args):
    import numpy as np
    import torch
    import paper_2005_07547_b200 as pb

    rank, world, local = dist_env()
    # PSTF_BENCH_BACKEND=gloo: the multi-rank code path on fewer GPUs than ranks (a test of
    # bench.py itself, collectives through the host; never a measurement)
    backend = os.environ.get("PSTF_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.force_sharded:
        import torch.distributed as dist
        if world == 1:  # a one-rank NCCL group exercises the multi-GPU code path on one GPU
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    W, H, B = args.width, args.height, args.bounces
    base = DIAMETER / 256.0
    mode = pb.MODE_ATOMIC if args.mode == "atomic" else pb.MODE_ORDERED
    stores = [pb.FieldStore(pb.FieldStoreConfig(kind=k, capacity_log2=args.capacity_log2,
                                                base_cell_size=base), device=local)
              for k in (pb.KIND_LO, pb.KIND_LO_MINUS_E, pb.KIND_FLI)]
    S = max(1, args.streams)
    drift = args.config == 5
    strong = world > 1 and args.scaling == "strong"
    n_paths = W * H
    p0, p1 = (n_paths * rank // world, n_paths * (rank + 1) // world) if strong else (0, n_paths)
    n = (p1 - p0) * B  # this rank's vertices per iteration
    # weak: rank r traces its own 1 spp of the frame (its own seed); strong: rank r traces the
    # image stripe [p0, p1) of the one frame (all bounces of its paths)
    seed = 0x5EED + (0 if strong else 7919 * rank)
    bufs = []
    for i in range(1 if drift else S):
        b, _ = pb.synth_generate(W, H, B, seed=seed, iteration=i, path0=p0, npaths=p1 - p0,
                                 scene=1 if args.config == 3 else 0)
        bufs.append(b)
    if drift:
        S = 1
    cv_out = None
    if args.config == 3:  # CV lookup at every vertex (estimators.cpp:453-462): RGB f64 + valid
        cv_out = (torch.empty((3, n), dtype=torch.float64, device="cuda"),
                  torch.empty(n, dtype=torch.uint8, device="cuda"))
    torch.cuda.synchronize()

    def regenerate(i):
        """config 5: the camera drifts +0.02 per iteration (untimed input production)"""
        shift = ((0.02 * i + 0.9) % 1.8) - 0.9
        pb.synth_generate(W, H, B, seed=seed, iteration=i, cam_shift_x=shift, out=bufs[0],
                          path0=p0, npaths=p1 - p0)
    sharded = None
    if dist is not None:
        # one field cache over the ranks: replicated stores, all-reduced accumulators
        from paper_2005_07547_b200.shard import Collectives, CudaBackend, ShardedFieldCache
        sharded = ShardedFieldCache(CudaBackend(stores, rank, world),
                                    Collectives(dist, torch.device("cuda", local)))

    def step(i):
        if sharded is not None:
            sharded.iteration((bufs[i % S], n))
            return
        if cv_out is not None:  # config 3: the CV lookup of every vertex fused into the pass
            pb.vertex_pass_cv(stores[0], stores[1], stores[2], None, bufs[i % S], n, mode=mode,
                              out=cv_out)
        else:
            pb.vertex_pass(stores[0], stores[1], stores[2], None, bufs[i % S], n, mode=mode)
        pb.end_frame_all(stores)

    for i in range(args.warmup):
        if drift:
            regenerate(i)
        step(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    touched0 = sum(s.stats()["touched_total"] for s in stores)
    reds0 = stores[0].stats()["reds_total"]
    l2_bytes = torch.cuda.get_device_properties(local).L2_cache_size  # cudaDevAttrL2CacheSize
    dropped0 = [s.stats()["dropped"] for s in stores]
    launches0 = pb.kernel_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pb.profile_collect()
    with ClockSampler(local) as clk:
        pb.profile_enable(True)
        torch.cuda.synchronize()
        if drift:  # per-step events: the input regeneration stays outside the timed region
            evs = []
            per_iter = []
            for i in range(args.steps):
                pb.profile_enable(False)
                regenerate(args.warmup + i)
                pb.profile_enable(True)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                step(args.warmup + i)
                e1.record()
                evs.append((e0, e1))
                pb.profile_enable(False)
                per_iter.append([(x["evicted_last"], x["dropped"], x["live"], x["new_keys_last"])
                                 for x in (s.stats() for s in stores)])  # untimed (events)
                pb.profile_enable(True)
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs)
        else:
            ev0.record()
            for i in range(args.steps):
                step(args.warmup + i)
            ev1.record()
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
        pb.profile_enable(False)
    launches = pb.kernel_launch_count() - launches0
    prof = pb.profile_collect()
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_vertices = (W * H * B if strong else n * world) * args.steps
    value = total_vertices / (ms / 1e3)
    ms_step = ms / args.steps
    st = [s.stats() for s in stores]

    # roofline: dominant kernel = the fused vertex pass (k_vertex_pass)
    peak, peak_src = peaks()
    vp = [(k.strip("()"), v) for k, v in prof.items() if "k_vertex_pass" in k]
    vp_ms, vp_n = (vp[0][1] if vp else (float("nan"), 1))
    vp_avg = vp_ms / max(vp_n, 1)
    cv_bytes = 25 * n if cv_out is not None else 0  # +25 B per CV lookup (config 3)
    vp_bytes = BYTES_PER_VERTEX * n + cv_bytes  # the CV outputs are written by the fused kernel
    ach = vp_bytes / (vp_avg / 1e3) / 1e9
    mean_touched = (sum(s["touched_total"] for s in st) - touched0) / args.steps
    # atomic roofline: fp64 RED element updates the fused kernel issued (after the
    # per-vertex aggregation) over its time, against this GPU's measured RED peak
    reds_step = (st[0]["reds_total"] - reds0) / args.steps
    red_peak = pb.red_peak(local)
    red_ach = reds_step / (vp_avg / 1e3) if reds_step else 0.0
    step_bytes = BYTES_PER_VERTEX * n + BYTES_PER_TOUCHED * mean_touched + cv_bytes
    step_ach = step_bytes / (ms_step / 1e3) / 1e9
    # DRAM traffic of the dominant kernel: not measurable inside this run (it needs an ncu
    # capture); the value comes from the committed capture named in traffic_source
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_vertex_pass_traffic.json")
    # the capture is of the config-2 ATOMIC tiled kernel; other kernels have none
    if os.path.exists(tpath) and args.mode == "atomic" and args.config == 2:
        try:
            with open(tpath) as f:
                tj = json.load(f)
            traffic = tj.get("dram_bytes_per_launch")
            traffic_src = ("past capture, not this run: profiles/ncu_vertex_pass_traffic.json (%s)"
                           % tj.get("source", "ncu --set full"))
        except Exception:
            traffic = None
    kernels = {k: {"ms_per_step": v[0] / args.steps, "launches": v[1]}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": DATA,
        "impl": "b200",
        "config": bench_config(args, S, world, multi=sharded is not None),
        "l2_bytes": l2_bytes,  # cudaDevAttrL2CacheSize (inputs per step are larger)
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "spec_peak": 8000.0, "frac_of_spec": ach / 8000.0,
                     "frac": ach / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": vp[0][0] if vp else None,
                     "bytes_per_launch": vp_bytes, "avg_launch_ms": vp_avg,
                     "peak_source": peak_src},
        "step_roofline": {"achieved": step_ach, "peak": peak, "unit": "GB/s",
                          "frac": step_ach / peak,
                          "bytes_per_step": step_bytes, "touched_cells_per_step": mean_touched},
        "atomic_roofline": {"bound": "l2_atomic", "achieved": red_ach / 1e9,
                            "peak": red_peak / 1e9, "unit": "Gop/s (fp64 RED elements)",
                            "frac": red_ach / red_peak if red_peak else None,
                            "reds_per_vertex": reds_step / n,
                            "peak_source": "pstf_diag_red_peak: 8 distinct L2-resident 32 B "
                                           "cells x 4 components per warp instruction"},
        "kernels": kernels,
        "field_stats": {k: [s[k] for s in st] for k in ("live", "dropped", "rejected",
                                                         "new_keys_last", "touched_last",
                                                         "placement_rounds_last")},
        "clocks": clk.summary(),
    }
    if drift:  # config 5 (probe-length stress): probe distances, drops and evictions
        ev = [[it[j][0] for it in per_iter] for j in range(3)]
        dr = [[it[j][1] for it in per_iter] for j in range(3)]
        line["probe_stress"] = {
            "capacity_log2": args.capacity_log2,
            "probe_hist_lo_loe_fli": [s.probe_histogram().tolist() for s in stores],
            "dropped_per_iteration": [(s["dropped"] - d0) / args.steps
                                      for s, d0 in zip(st, dropped0)],
            "evicted_total_lo_loe_fli": [sum(e) for e in ev],
            "iterations_with_evictions": [sum(1 for x in e if x) for e in ev],
            "evicted_per_iteration_fli": ev[2],
            "dropped_cumulative_fli": dr[2],
            "live_per_iteration_fli": [it[2][2] for it in per_iter],
            "new_keys_per_iteration_fli": [it[2][3] for it in per_iter],
            "load_factor": [s["live"] / float(1 << args.capacity_log2) for s in st],
        }

    # e2e: same metric through the C ABI with pinned HOST vertex arrays (H2D every step)
    if not args.no_e2e:
        hosts = [bufs[i].cpu().pin_memory() for i in range(min(2, S))]
        E = max(1, args.e2e_steps)

        def estep(i):
            if sharded is not None:  # H2D of this rank's stream, then the sharded iteration
                bufs[0].copy_(hosts[i % len(hosts)], non_blocking=True)
                sharded.iteration((bufs[0], n))
            else:
                pb.vertex_pass_host(stores[0], stores[1], stores[2], None, hosts[i % len(hosts)],
                                    n, mode=mode)
                pb.end_frame_all(stores)
            return [s.stats()["live"] for s in stores]  # D2H read of the step's result

        estep(0)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(E):
            estep(i + 1)
        torch.cuda.synchronize()
        et = time.perf_counter() - t0
        if dist:
            t = torch.tensor([et], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            et = float(t.item())
        line["e2e"] = {"value": (W * H * B if strong else n * world) * E / et, "unit": UNIT,
                       "h2d_bytes_per_step": BYTES_PER_VERTEX * n,
                       "d2h_bytes_per_step": 3 * 8 * 11, "steps": E,
                       "path": ("pstf_vertex_pass_host (pinned host SoA, chunked H2D overlapped "
                                "with phase 1) + pstf_fields_end_frame + stats readback")
                       if sharded is None else
                       "pinned host SoA -> HBM copy + multi-GPU iteration + stats readback"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference_run(args, 2, 1, budget_s=args.cpu_seconds)
            line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                       "host", "phases_ms_per_iteration")}
        except Exception as e:  # report, never fail the GPU line
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                                    "sample": f"error: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def spawn_ranks(args):
    """`--gpus N` without a launcher: re-run this command as N ranks (one process per GPU) under
    torch.distributed.run on this node; rank 0's JSON line is the output"""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus and not (world == 1 and args.gpus == 1):
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())

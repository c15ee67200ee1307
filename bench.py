"""bench.py -- GCDF value+grad queries/s with active-set detection on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--precision fp16|bf16|fp32|fp16x3|bf16x3]
    python bench.py --impl reference ...      # the float64 CPU oracle on host cores

One step = one SCO iteration of the hot path (all SURVEY §8(a) rows): an incremental
scene update (A9: 200 removes + 200 adds on a moved box) followed by the fused
detect over every (waypoint, live point) pair (A2-A8) with the count read back on the
host; at N > 1 the points are sharded by rank and every rank's detect call returns the
gathered active set (the library's NCCL all-gather group + merge kernel on the call's
stream).  `--gpus N` without WORLD_SIZE re-launches itself under torch.distributed.run
with N ranks; under a launcher WORLD_SIZE must equal --gpus.  `value` counts every (waypoint, live point) pair of the whole
job per second.  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import synth  # noqa: E402

METRIC = "GCDF value+grad queries/sec (with active-set detection)"
FLOPS_PAIR_TOTAL = {128: 333_312, 32: 21_888, 256: 1_321_984}   # fwd 167,168 + bwd 166,144 (H=128)
FLOPS_PAIR_TENSOR = {128: 327_680, 32: 20_480, 256: 1_310_720}   # the ten H x H GEMMs (tensor-eligible)
ACT = {"relu": 1, "softplus": 2}                   # MLPW activation ids (R9, R26)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--precision", default="auto", choices=["auto", "fp16", "bf16", "fp32", "fp16x3", "bf16x3"])
    ap.add_argument("--hidden", type=int, default=None, choices=[128, 256],
                    help="hidden width override for the H = 128 configs (256: NEXT-4 variant, DESIGN.md R27)")
    ap.add_argument("--activation", default="relu", choices=["relu", "softplus"],
                    help="hidden activation of the random-init network (softplus: NEXT-4 variant, DESIGN.md R26)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--partition-radius", type=float, default=1.8,
                    help="also time the range-partitioned detect (NEXT-1) at this radius; 0 = skip")
    ap.add_argument("--no-kernels", dest="kernels", action="store_false",
                    help="skip the standalone K1 / K3 HBM measurements of the default run")
    ap.add_argument("--no-workloads", dest="workloads", action="store_false",
                    help="skip the C2 / C3 / C4 measurements of the default run")
    ap.add_argument("--no-variants", dest="variants", action="store_false",
                    help="skip the softplus / H = 256 variant measurements (NEXT-4) of the default run")
    ap.add_argument("--latency-calls", type=int, default=50,
                    help="detect-latency sample size (wall time q on device -> count on host); 0 = skip")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "host"],
                    help="exchange backend at N > 1: nccl (product) or host (TEST backend: gloo all-gather "
                         "on the host, for the dry run of the N > 1 path on one GPU)")
    ap.add_argument("--same-device", action="store_true",
                    help="DRY RUN: every rank on cuda:0 (needs --comm host); the line is marked dry_run")
    return ap.parse_args()


def relaunch_under_torchrun(a):
    """--gpus N > 1 without a launcher: run this script under torch.distributed.run."""
    import socket
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


# ----------------------------------------------------------------------------- oracle timing
def cpu_oracle_rate(cfg, pts, q, sample_pts=8192, nthreads=None, seed=12345, single_thread=False, act=1, hidden=None):
    """The oracle as it stands on the host cores: detect over a bounded sample of the
    workload -- one waypoint row per core (the oracle threads over waypoint rows) x
    sample_pts points."""
    import oracle
    nthreads = nthreads or os.cpu_count() or 1
    m = oracle.MLP(synth.weights_path(cfg.H, act=act))
    tau = synth.load_tau(cfg.name, act, hidden)
    rng = np.random.default_rng(seed)
    qs = q.reshape(-1, 9)
    wsel = np.sort(rng.choice(qs.shape[0], size=min(nthreads, qs.shape[0]), replace=False))
    psel = np.sort(rng.choice(pts.shape[0], size=min(sample_pts, pts.shape[0]), replace=False))
    used = min(nthreads, len(wsel))
    t0 = time.perf_counter()
    m.detect(pts[psel], psel.astype(np.int64), qs[wsel], synth.inputs.DELTA, tau, nthreads=used)
    dt = time.perf_counter() - t0
    n = len(wsel) * len(psel)
    r = {"value": n / dt, "unit": "queries/s", "cores": int(used), "kind": "oracle", "pairs": n, "seconds": dt,
         "sample": f"{len(wsel)} waypoints x {len(psel)} points of {cfg.name} ({n} pairs, "
                   f"float64 detect incl. gradients, one waypoint row per thread), {dt:.1f} s"}
    if single_thread:
        p1 = psel[: max(1, len(psel) // 8)]
        t0 = time.perf_counter()
        m.detect(pts[p1], p1.astype(np.int64), qs[wsel[:1]], synth.inputs.DELTA, tau, nthreads=1)
        d1 = time.perf_counter() - t0
        r["single_thread"] = {"value": len(p1) / d1, "pairs": len(p1), "seconds": d1}
    return r


def run_reference(a):
    """--impl reference: the float64 oracle (this tier's reference arm) on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = synth.get_config(a.config)
    hidden = a.hidden if a.hidden and a.hidden != cfg.H else None
    if hidden:
        cfg = dataclasses.replace(cfg, H=hidden)
    pts, _ = synth.make_scene_points(cfg)
    q = synth.make_waypoints(cfg)
    times, n_pairs, r = [], 0, None
    for i in range(a.warmup + a.steps):
        r = cpu_oracle_rate(cfg, pts, q, sample_pts=2048 if cfg.H <= 128 else 512, seed=1000 + i,
                            act=ACT[a.activation], hidden=hidden)
        if i >= a.warmup:
            times.append(r["seconds"])
            n_pairs += r["pairs"]
    total = sum(times)
    v = n_pairs / total
    sample = f"each step: one waypoint row per core x 2048 points of {cfg.name} ({r['pairs']} pairs)"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "queries/s", "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * total / a.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.desc}; {sample}"},
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": r["cores"], "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        relaunch_under_torchrun(a)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != a.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {a.gpus}: launch one rank per GPU "
                 f"(torchrun --nproc-per-node {a.gpus} bench.py --gpus {a.gpus})")
    if a.same_device and a.comm != "host":
        sys.exit("bench.py: --same-device (dry run) needs --comm host (one GPU cannot host two NCCL ranks)")
    import torch
    import torch.distributed as dist
    from paper_2601_18548_b200 import BF16, BF16X3, FP16, FP16X3, FP32, Context
    from paper_2601_18548_b200.gcdf import load_library

    rank = int(os.environ.get("RANK", "0"))
    local = 0 if a.same_device else int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        if a.comm == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    red_dev = "cpu" if (world > 1 and a.comm == "host") else None  # where max-over-ranks reductions run
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    lib = load_library()
    prec = a.precision
    cfg = synth.get_config(a.config)
    hidden = a.hidden if a.hidden and a.hidden != cfg.H else None
    if hidden:
        cfg = dataclasses.replace(cfg, H=hidden)
    if prec == "auto":  # the tensor-core path needs H = 128 (C1's H = 32 net runs on the fp32 path)
        prec = "fp16" if lib.gcdf_has_tcgen05() and cfg.H >= 128 else "fp32"
    act = ACT[a.activation]
    tau = synth.load_tau(cfg.name, act, hidden)
    delta = synth.inputs.DELTA
    pts, boxes = synth.make_scene_points(cfg)
    q_np = synth.make_waypoints(cfg)
    n_wp = cfg.B * cfg.N
    slack = 4096
    max_active = int(min(cfg.pairs // world + 1024, max(4 * cfg.pairs // 100 // world, 1 << 16)))
    ctx = Context(local, precision={"fp16": FP16, "bf16": BF16, "fp32": FP32, "fp16x3": FP16X3, "bf16x3": BF16X3}[prec], scene_capacity=cfg.M + slack,
                  max_waypoints=n_wp, max_active=max_active, rank=rank, world=world,
                  max_candidates=(cfg.pairs // world + 4096) if a.partition_radius > 0 else 0)
    ctx.load_weights(synth.weights_path(cfg.H, act=act))
    ctx.update_scene(pts)
    if world > 1:
        if a.comm == "nccl":
            ctx.dist_init()   # NCCL communicator inside the library (id broadcast by torch.distributed)
        else:
            def gloo_allgather(send, recv):
                n_ = send.shape[0]
                parts = [torch.empty(n_, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(parts, torch.from_numpy(send.copy()))
                for r_ in range(world):
                    recv[r_ * n_:(r_ + 1) * n_] = parts[r_].numpy()
            ctx.dist_init_host(gloo_allgather)
    q = torch.from_numpy(q_np).to(dev)
    # output capacity of the (gathered) result; at N > 1 it also sets the exchange stride
    # (ceil(capacity / N) records per rank), so after the first warm-up step it is the
    # observed count + 10 % (the scene updates move it by ~0.01 %)
    cap = [max_active * world]
    outs = ctx.alloc_detect_outputs(n_wp, max_active * world)
    # Scene-update inputs of every step (A9: 200 removes + 200 adds of a moved box), made
    # before any clock starts: adds are points of a randomly moved clutter box, removals
    # disjoint sets of the initially live ids (valid whatever ids the adds reuse).
    e2e_steps = a.e2e_steps or max(1, a.steps)  # (as many steps as the device-timed region: the same thermal / power-cap window length)
    n_upd = a.warmup + a.steps + e2e_steps
    gen = np.random.default_rng([cfg.seed, 7])
    n_chg = int(max(1, min(200, cfg.M // (2 * n_upd))))  # 200 (C4 dynamics) unless the scene is tiny
    adds = [synth.inputs.scene_update_batch(gen, boxes, np.zeros((0, 3)), n_add=n_chg)[0] for _ in range(n_upd)]
    rems = list(gen.choice(cfg.M, size=(n_upd, n_chg), replace=False))
    upd_i = [0]

    def scene_step():
        i = upd_i[0]
        upd_i[0] += 1
        ctx.update_scene(adds[i], rems[i])
        return adds[i], rems[i]

    def step():
        scene_step()
        # no host sync inside the device-timed step (the count is read after the timed
        # region); at N > 1 the exchange runs on the call's stream inside the library
        o = ctx.detect_active_set(q, delta, tau, outputs=outs, capacity=cap[0], sync_count=False)
        return o

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=red_dev or dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # L2 flush buffer (> 126 MB L2) written between timed steps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for i in range(a.warmup):
        o = step()
        if i == 0:
            n0 = int(o["count"].item())
            cap[0] = min(max_active * world, world * (int(1.1 * n0 / world) + 2048))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ctx.profile_enable(True)
    ctx.profile_read(reset=True)
    l0 = ctx.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    n_live_total = 0
    last = None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(a.steps):
        flush.zero_()
        ev[i][0].record()
        last = step()
        ev[i][1].record()
        n_live_total += ctx.scene_info()["n_live"]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.launches - l0
    mlp_ms, mlp_n = ctx.profile_read(reset=True)
    x_ms, x_n = ctx.profile_read_exchange(reset=True)
    ctx.profile_enable(False)
    clk = clocks.stop()
    t_ms = sum(s.elapsed_time(e) for s, e in ev)
    t_max = max_over_ranks(t_ms)
    # n_live is the global live count (the id rule is replicated on every rank)
    pairs_total = n_live_total * n_wp           # every (waypoint, live point) pair of the job
    value = pairs_total / (t_max / 1e3)
    n_active = int(last["count"].item())
    exchange = None
    if world > 1:
        exchange = {"backend": ctx.dist_info(), "ms_per_step": (x_ms / x_n) if x_n else None,
                    "share_of_step": (x_ms / t_ms) if (x_n and t_ms > 0) else None,
                    "capacity": cap[0], "stride_records_per_rank": -(-cap[0] // world),
                    "bytes_received_per_rank": (world - 1) * (48 * -(-cap[0] // world) + 8 * (2 * n_wp + 1)),
                    "what": "all-gather group (headers + records) + merge kernel, CUDA events on the call's stream"}

    # roofline of the dominant kernel (fused MLP): algorithmic flops per launch / live duration
    peaks, peak_src = measured_peaks()
    local_pairs = n_wp * (n_live_total / a.steps) / world
    if prec in ("bf16", "fp16", "fp16x3", "bf16x3"):
        # algorithmic flops: the method's ten H x H GEMMs per pair; fp16x3 (K2c)
        # executes each of them 3 times (the split, R25): reported as a side field
        n_terms = 3 if prec in ("fp16x3", "bf16x3") else 1
        flops = FLOPS_PAIR_TENSOR[cfg.H] * local_pairs
        achieved = flops / (mlp_ms / mlp_n / 1e3) / 1e12
        # peak: the measured BURST dense figure (the higher, stricter one) whatever the length of
        # the timed region; the fraction of the sustained figure is a side field.  fp16 and bf16
        # share the same dense tensor peak on B200 (nominal 2.25 PFLOP/s each)
        peak = float(peaks.get("bf16_tflops"))
        peak_s = float(peaks.get("bf16_tflops_sustained", peak))
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "frac_of_sustained_peak": achieved / peak_s,
                "traffic": None, "peak_source": f"{peak_src} bf16_tflops (MEASURED_PEAKS.json burst; fp16 dense = bf16 dense)",
                "kernel": ("k_mlp_tc3" if n_terms == 3 else "k_mlp_tc_sp" if act == 2 else
                           "k_mlp_tc_wide" if cfg.H == 256 else "k_mlp_tc") +
                          " (fused transform + MLP fwd/bwd + threshold/min/compaction)",
                "kernel_ms_avg": mlp_ms / mlp_n, "flops_per_pair": FLOPS_PAIR_TENSOR[cfg.H]}
        if n_terms > 1:
            roof["executed_flops_per_pair"] = n_terms * FLOPS_PAIR_TENSOR[cfg.H]
            roof["executed_frac"] = n_terms * achieved / peak
    else:
        sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
        peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12   # FP32 FFMA: 148 SMs x 128 lanes x 2 flops x clock
        flops = FLOPS_PAIR_TOTAL[cfg.H] * local_pairs
        achieved = flops / (mlp_ms / mlp_n / 1e3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": None, "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 x sm_max_mhz",
                "kernel": "k_mlp_simt (fused transform + MLP fwd/bwd + threshold/min/compaction)",
                "kernel_ms_avg": mlp_ms / mlp_n, "flops_per_pair": FLOPS_PAIR_TOTAL[cfg.H]}
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists() and prec in ("bf16", "fp16") and act == 1 and cfg.H == 128:  # (measured for k_mlp_tc only)
        t = json.loads(tf.read_text()).get("k_mlp_tc")
        if t:
            roof["traffic"] = t["bytes"]
            roof["traffic_source"] = t["source"]
            roof["algorithmic_dram_bytes"] = int(16 * cfg.M + 48 * n_active + 8 * local_pairs / 128)
    kshare = mlp_ms / t_ms if t_ms > 0 else None

    # e2e through the public API with host buffers: each step = the scene update (host
    # arrays in) + the host-buffer detect call (q in from pinned host memory, records /
    # offsets / min / argmin out to pinned host memory; the library does the copies).
    q_pin = torch.from_numpy(q_np).pin_memory()
    host_out = ctx.alloc_host_outputs(n_wp, cap[0], pinned=True)
    h2d = d2h = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_pairs = 0
    for i in range(e2e_steps):
        add_i, rem_i = scene_step()
        o = ctx.detect_active_set_host(q_pin, delta, tau, host_out)
        n = int(o["n"])
        h2d += q_pin.numel() * 4 + add_i.nbytes + rem_i.nbytes
        d2h += n * 48 + host_out["wp_offsets"].numel() * 8 + host_out["wp_min"].numel() * 4 + \
            host_out["wp_argmin"].numel() * 8 + 8
        e2e_pairs += ctx.scene_info()["n_live"] * n_wp
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)

    # NEXT-1: the range-partitioned detect on the same workload (device time per call)
    part = None
    if a.partition_radius > 0 and world == 1:
        for _ in range(3):
            ctx.detect_active_set_partitioned(q, a.partition_radius, delta, tau, outputs=outs, sync_count=False)
        torch.cuda.synchronize()
        k = max(3, a.steps)
        pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        ctx.profile_read(reset=True)
        ctx.profile_enable(True)
        for i in range(k):
            flush.zero_()
            pe[i][0].record()
            po = ctx.detect_active_set_partitioned(q, a.partition_radius, delta, tau, outputs=outs, sync_count=False)
            pe[i][1].record()
        torch.cuda.synchronize()
        p_mlp_ms, p_mlp_n = ctx.profile_read(reset=True)
        ctx.profile_enable(False)
        p_ms = sum(s_.elapsed_time(e_) for s_, e_ in pe) / k
        p_pairs = int(po["part_sizes"].sum().item())
        n_live = ctx.scene_info()["n_live"]
        part = {"radius_m": a.partition_radius, "ms_per_step": p_ms, "pairs_per_step": p_pairs,
                "pairs_fraction": p_pairs / (n_live * n_wp), "active_per_step": int(po["count"].item()),
                "evaluated_pairs_per_s": p_pairs / (p_ms / 1e3),
                "covered_pairs_per_s": n_live * n_wp / (p_ms / 1e3),
                "mlp_kernel_ms": p_mlp_ms / max(p_mlp_n, 1),
                "what": "detect over I_{M,i} (points within radius of each step's base, PAPER.md:401); "
                        "covered = all B*N*M pairs of the step served by one partitioned call"}

    # active-set detect latency per SCO iteration = wall time of one detect
    # call from q resident on the device to the count on the host (collectives included),
    # p50 / p99 over `latency_calls` calls after 5 warm-ups
    lat = None
    if a.latency_calls > 0:
        for _ in range(5):
            ctx.detect_active_set(q, delta, tau, outputs=outs, capacity=cap[0], sync_count=True)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.latency_calls):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            ctx.detect_active_set(q, delta, tau, outputs=outs, capacity=cap[0], sync_count=True)
            ts.append(time.perf_counter() - t0)
        tt = torch.tensor(ts, device=red_dev or dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = np.sort(tt.cpu().numpy()) * 1e3
        lat = {"p50_ms": float(np.percentile(ms, 50)), "p99_ms": float(np.percentile(ms, 99)),
               "calls": a.latency_calls, "what": "wall time, q on device -> active count on host"}
        if world == 1:  # the same call chain replayed as a captured CUDA graph
            for name, r in (("graph", 0.0), ("graph_partitioned", a.partition_radius)):
                if name == "graph_partitioned" and r <= 0:
                    continue
                g = ctx.detect_graph(q, delta, tau, radius=r, capacity=max_active)
                for _ in range(5):
                    g.launch()
                ts = []
                for _ in range(a.latency_calls):
                    t0 = time.perf_counter()
                    g.launch()
                    ts.append(time.perf_counter() - t0)
                g.close()
                ms = np.sort(np.array(ts)) * 1e3
                lat[name] = {"p50_ms": float(np.percentile(ms, 50)), "p99_ms": float(np.percentile(ms, 99))}

    # NEXT-4 variants on the same workload (single GPU, default run only): device time per
    # detect over the whole scene with the softplus network (K2s), the H = 256 network (K2w),
    # the split paths (K2c) and the fp32 SIMT parity path (K2f), each in a context of its own;
    # tensor roofline against the same peak (K2f: the FP32-ALU peak)
    variants = None
    if world == 1 and a.variants and a.activation == "relu" and not hidden and prec == "fp16":
        variants = {}
        for name, act_v, h_v, prec_v in (("softplus", 2, None, FP16), ("hidden256", 1, 256, FP16),
                                         ("fp16x3", 1, None, FP16X3), ("bf16x3", 1, None, BF16X3),
                                         ("fp32", 1, None, FP32)):
            cfg_v = dataclasses.replace(cfg, H=h_v) if h_v else cfg
            ctx_v = Context(local, precision=prec_v, scene_capacity=cfg.M + slack, max_waypoints=n_wp,
                            max_active=max_active)
            ctx_v.load_weights(synth.weights_path(cfg_v.H, act=act_v))
            ctx_v.update_scene(pts)
            tau_v = synth.load_tau(cfg.name, act_v, h_v)
            outs_v = ctx_v.alloc_detect_outputs(n_wp, max_active)
            for _ in range(2):
                ctx_v.detect_active_set(q, delta, tau_v, outputs=outs_v, sync_count=False)
            torch.cuda.synchronize()
            ctx_v.profile_read(reset=True)
            ctx_v.profile_enable(True)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
            for e0, e1 in evs:
                flush.zero_()
                e0.record()
                ov = ctx_v.detect_active_set(q, delta, tau_v, outputs=outs_v, sync_count=False)
                e1.record()
            torch.cuda.synchronize()
            k_ms, k_n = ctx_v.profile_read(reset=True)
            ctx_v.profile_enable(False)
            ms_v = sum(e0.elapsed_time(e1) for e0, e1 in evs) / len(evs)
            pairs_v = ctx_v.scene_info()["n_live"] * n_wp
            simt = prec_v == FP32  # (the fp32 SIMT parity path K2f: FP32-ALU roofline)
            ach = (FLOPS_PAIR_TOTAL if simt else FLOPS_PAIR_TENSOR)[cfg_v.H] * pairs_v / (k_ms / k_n / 1e3) / 1e12
            pk = (148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12 if simt
                  else float(peaks.get("bf16_tflops")))
            split = prec_v in (FP16X3, BF16X3)
            variants[name] = {"kernel": "k_mlp_simt" if simt else "k_mlp_tc_sp" if act_v == 2 else "k_mlp_tc3" if split
                              else "k_mlp_tc_wide", "hidden": cfg_v.H,
                              "activation": "softplus" if act_v == 2 else "relu", "ms_per_step": ms_v,
                              "precision": ("fp16x3 (fp32-accurate split, R25)" if prec_v == FP16X3 else
                                            "bf16x3 (3-term split bf16, R29)" if prec_v == BF16X3 else
                                            "fp32 (SIMT parity path)" if simt else "fp16"),
                              "value": pairs_v / (ms_v / 1e3), "unit": "queries/s", "tau": tau_v,
                              "active_per_step": int(ov["count"].item()),
                              "roofline": {"bound": "alu" if simt else "tensor", "achieved": ach, "peak": pk,
                                           "unit": "TFLOP/s", "frac": ach / pk,
                                           "flops_per_pair": (FLOPS_PAIR_TOTAL if simt else FLOPS_PAIR_TENSOR)[cfg_v.H]}}
            if split:
                variants[name]["roofline"].update(executed_flops_per_pair=3 * FLOPS_PAIR_TENSOR[cfg_v.H],
                                                  executed_frac=3 * ach / pk)
            ctx_v.close()
            del outs_v
            torch.cuda.empty_cache()

    # the HBM-bound standalone stages on the same workload: K1 pair generation +
    # base-frame transform (16 B written per pair, points read once) and K3 threshold + min +
    # compaction over the dense values / gradients of one query (4 B read per pair + 36 B
    # gradient read + 48 B record written per active).  Device time per call (CUDA events,
    # L2 flushed before each), achieved algorithmic GB/s vs the measured copy bandwidth.
    kernels = None
    if world == 1 and a.kernels:
        kernels = {}
        hbm = float(peaks.get("hbm_gbs"))
        lbnd = ctx.scene_info()["local_bound"]
        n_live = ctx.scene_info()["n_live"]

        def time_calls(fn, k=5):
            fn()
            torch.cuda.synchronize()
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
            for e0, e1 in evs:
                flush.zero_()
                e0.record()
                fn()
                e1.record()
            torch.cuda.synchronize()
            return sorted(e0.elapsed_time(e1) for e0, e1 in evs)[k // 2]
        pg = torch.empty((n_wp, lbnd, 4), dtype=torch.float32, device=dev)
        ms1 = time_calls(lambda: ctx.pairgen_transform(q, out=pg))
        b1 = 16 * n_wp * lbnd + 16 * lbnd
        kernels["k1_pairgen_transform"] = {"ms": ms1, "algorithmic_bytes": b1, "achieved_gbs": b1 / ms1 / 1e6,
                                           "peak_gbs": hbm, "frac": b1 / ms1 / 1e6 / hbm,
                                           "bytes_per_unit": "16 B written per (waypoint, slot) pair + 16 B per slot read"}
        del pg
        vals, grs = ctx.query_values_grads(q)
        outs_k = ctx.alloc_detect_outputs(n_wp, max_active)
        ms3 = time_calls(lambda: ctx.compact_dense(vals, grs, delta, tau, outputs=outs_k, sync_count=False))
        n3 = int(outs_k["count"].item())
        b3 = 4 * n_wp * lbnd + n3 * (36 + 48)
        kernels["k3_compact_dense"] = {"ms": ms3, "algorithmic_bytes": b3, "achieved_gbs": b3 / ms3 / 1e6,
                                       "peak_gbs": hbm, "frac": b3 / ms3 / 1e6 / hbm, "active": n3,
                                       "live_pairs": n_live * n_wp,
                                       "bytes_per_unit": "4 B value read per pair + (36 B gradient read + 48 B record "
                                                         "written) per active"}
        del vals, grs, outs_k
        torch.cuda.empty_cache()

    # the other configurations of BASELINE.json on the same GPU (default run only): C4 is the
    # batched-replanning workload (128 trajectories x 64 waypoints, 20k points, 200 + 200 scene
    # updates per step), C2 / C3 the single-trajectory latency cases.  Per config: device time
    # per SCO step (scene update + fused detect, L2 flushed before each) and the wall-time
    # latency of one detect call (q on device -> count on host) replayed as a CUDA graph.
    workloads = None
    if world == 1 and a.workloads and a.config == "C5" and prec == "fp16" and not hidden and a.activation == "relu":
        workloads = {}
        for wname in ("C2", "C3", "C4"):
            wc = synth.get_config(wname)
            wpts, wboxes = synth.make_scene_points(wc)
            wq = torch.from_numpy(synth.make_waypoints(wc)).to(dev)
            wn = wc.B * wc.N
            wma = int(min(wc.pairs + 1024, max(4 * wc.pairs // 100, 1 << 16)))
            wctx = Context(local, precision=FP16, scene_capacity=wc.M + slack, max_waypoints=wn, max_active=wma)
            wctx.load_weights(synth.weights_path(wc.H))
            wctx.update_scene(wpts)
            wtau = synth.load_tau(wname)
            wouts = wctx.alloc_detect_outputs(wn, wma)
            wgen = np.random.default_rng([wc.seed, 11])
            wk = 5
            wch = int(max(1, min(200, wc.M // (2 * (wk + 2)))))
            wadd = [synth.inputs.scene_update_batch(wgen, wboxes, np.zeros((0, 3)), n_add=wch)[0] for _ in range(wk + 2)]
            wrem = list(wgen.choice(wc.M, size=(wk + 2, wch), replace=False))
            for i in range(2):
                wctx.update_scene(wadd[i], wrem[i])
                wctx.detect_active_set(wq, delta, wtau, outputs=wouts, sync_count=False)
            torch.cuda.synchronize()
            wev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(wk)]
            wpairs = 0
            for i, (e0, e1) in enumerate(wev):
                flush.zero_()
                e0.record()
                wctx.update_scene(wadd[2 + i], wrem[2 + i])
                wo = wctx.detect_active_set(wq, delta, wtau, outputs=wouts, sync_count=False)
                e1.record()
                wpairs += wctx.scene_info()["n_live"] * wn
            torch.cuda.synchronize()
            wms = sum(e0.elapsed_time(e1) for e0, e1 in wev) / wk
            g = wctx.detect_graph(wq, delta, wtau, capacity=wma)
            for _ in range(5):
                g.launch()
            ts = []
            for _ in range(20):
                t0 = time.perf_counter()
                g.launch()
                ts.append(time.perf_counter() - t0)
            g.close()
            workloads[wname] = {"desc": wc.desc, "ms_per_step": wms, "value": wpairs / wk / (wms / 1e3),
                                "unit": "queries/s", "active_per_step": int(wo["count"].item()),
                                "scene_update_per_step": f"{wch} removes + {wch} adds",
                                "detect_latency_graph_p50_ms": float(np.median(ts) * 1e3)}
            wctx.close()
            del wouts
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_oracle_rate(cfg, pts, q_np, sample_pts=65536 if cfg.H <= 128 else 16384, single_thread=True,
                              act=act, hidden=hidden)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": t_max / a.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": prec, "data": "synthetic (seeded clutter clouds + random-init weights)",
            "config": {"workload": f"{cfg.name}: {cfg.desc}", "B": cfg.B, "N": cfg.N, "points": cfg.M,
                       "hidden": cfg.H, "activation": a.activation, "pairs_per_step": int(pairs_total / a.steps), "delta": delta, "tau": tau,
                       "active_per_step": n_active, "scene_update_per_step": f"{n_chg} removes + {n_chg} adds",
                       "parallelism": f"points sharded over {world} GPU(s)",
                       "l2": "256 MiB buffer written between timed steps (L2 flush)"},
            "roofline": roof, "mlp_kernel_share_of_step": kshare, "exchange": exchange,
            "detect_latency": lat,
            "partitioned": part,
            "variants": variants,
            "kernels": kernels,
            "workloads": workloads,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_pairs / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": h2d // e2e_steps,
                    "d2h_bytes_per_step": d2h // e2e_steps, "steps": e2e_steps},
            "gpu_launches": launches, "clocks": clk,
        }
        if a.same_device:
            line["dry_run"] = ("all ranks on cuda:0 with the host test exchange backend: checks the N > 1 "
                               "code path, NOT a measurement")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

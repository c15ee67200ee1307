"""HBM-bound stages measured standalone on the bench workload (default C5), with CUDA events.

    python tools/hbm_bench.py [--config C5] [--reps 5] > gpurun_out/hbm.json

K1 gcdf_pairgen_transform: writes p' = (p_x - q_x, p_y - q_y, p_z, live) for every pair:
   algorithmic bytes = 16 B x pairs written + 16 B x points read.
K3 gcdf_compact_dense: threshold + per-waypoint min + compaction over a dense value array:
   algorithmic bytes = 4 B x pairs (values) + active x (36 B gradient read + 48 B staging
   write + 48 B staging read + 48 B record write) + 8 B x tiles (meta write + read).
Dense query (gcdf_query_values_grads) output: 40 B x pairs written (reported for context;
that kernel is tensor-bound).  Peaks: MEASURED_PEAKS.json hbm_gbs (copy, read + write).
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import synth  # noqa: E402
from paper_2601_18548_b200 import FP16, Context  # noqa: E402


def timed(fn, reps, flush):
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = synth.get_config(a.config)
    pts, _ = synth.make_scene_points(cfg)
    q = torch.from_numpy(synth.make_waypoints(cfg)).cuda()
    tau = synth.load_tau(cfg.name)
    n_wp = cfg.B * cfg.N
    ctx = Context(0, precision=FP16, scene_capacity=cfg.M + 4096, max_waypoints=n_wp, max_active=1 << 24)
    ctx.load_weights(synth.weights_path(cfg.H))
    ctx.update_scene(pts)
    lb = ctx.scene_info()["local_bound"]
    pairs = n_wp * lb
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {"config": cfg.name, "pairs": pairs, "hbm_peak_gbs": hbm,
           "hbm_peak_source": "measured" if peaks else "fallback"}

    pg = torch.empty((n_wp, lb, 4), dtype=torch.float32, device="cuda")
    ctx.pairgen_transform(q, pg)
    ms = timed(lambda: ctx.pairgen_transform(q, pg), a.reps, flush)
    b = 16 * pairs + 16 * lb
    out["K1_pairgen"] = {"ms": ms, "bytes": b, "GBps": b / ms / 1e6, "frac": b / ms / 1e6 / hbm}
    del pg

    v, g = ctx.query_values_grads(q)
    torch.cuda.synchronize()
    ms_q = timed(lambda: ctx.query_values_grads(q, values=v, grads=g), max(2, a.reps // 2), flush)
    out["dense_query"] = {"ms": ms_q, "bytes_written": 40 * pairs, "GBps_written": 40 * pairs / ms_q / 1e6}
    outs = ctx.alloc_detect_outputs(n_wp, 1 << 24)
    r = ctx.compact_dense(v, g, synth.inputs.DELTA, tau, outputs=outs)
    n_act = r["n"]
    ms = timed(lambda: ctx.compact_dense(v, g, synth.inputs.DELTA, tau, outputs=outs), a.reps, flush)
    tiles = pairs // 128
    b = 4 * pairs + n_act * (36 + 48 + 48 + 48) + 8 * 2 * tiles
    out["K3_compact_dense"] = {"ms": ms, "active": n_act, "bytes": b, "GBps": b / ms / 1e6,
                               "frac": b / ms / 1e6 / hbm,
                               "note": "3 finalize launches included (tile scan + ordered scatter)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""K3 standalone compaction probe (C5 by default): time gcdf_compact_dense over the dense
values / gradients of one query (L2 flushed before each call) and check it against a
torch filter of the same values (count, order, values, gradients, offsets)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import synth  # noqa: E402
from paper_2601_18548_b200 import FP16, Context, records_to_dict  # noqa: E402

cfg = synth.get_config(sys.argv[1] if len(sys.argv) > 1 else "C5")
pts, _ = synth.make_scene_points(cfg)
q = torch.from_numpy(synth.make_waypoints(cfg)).cuda()
tau = synth.load_tau(cfg.name)
ctx = Context(0, precision=FP16, scene_capacity=cfg.M + 4096, max_waypoints=cfg.B * cfg.N, max_active=1 << 22)
ctx.load_weights(synth.weights_path(cfg.H))
ctx.update_scene(pts)
v, g = ctx.query_values_grads(q)
outs = ctx.alloc_detect_outputs(cfg.B * cfg.N, 1 << 22)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ms = []
for i in range(8):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.compact_dense(v, g, synth.inputs.DELTA, tau, outputs=outs, sync_count=False)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
n = int(outs["count"].item())
act = (v - synth.inputs.DELTA) <= tau
idx = act.nonzero()
assert idx.shape[0] == n, (idx.shape[0], n)
rec = records_to_dict(outs["records"], n)
assert torch.equal(rec["wp"].long(), idx[:, 0]), "wp order"
lb = ctx.scene_info()["local_bound"]
assert torch.equal(rec["pt"].long(), idx[:, 1]), "pt order"   # world 1: global id = slot
assert torch.equal(rec["value"], v[idx[:, 0], idx[:, 1]])
assert torch.equal(rec["grad"], g[idx[:, 0], idx[:, 1]])
offs = torch.zeros(v.shape[0] + 1, dtype=torch.int64, device="cuda")
offs[1:] = torch.cumsum(act.sum(1), 0)
assert torch.equal(outs["wp_offsets"], offs)
alg = 4 * v.shape[0] * lb + n * (36 + 48)
best = sorted(ms)[len(ms) // 2]
print(f"K3 {cfg.name}: {n} actives, median {best:.3f} ms (all {['%.3f' % x for x in ms]}), "
      f"{alg / best / 1e6:.0f} GB/s algorithmic; parity vs torch filter OK")

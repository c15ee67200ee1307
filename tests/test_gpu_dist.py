"""The sharded detect's exchange inside the library on
the GPU, through the C ABI.

* NCCL backend at world 1 (gcdf_options.exchange, a one-rank communicator): the whole
  exchange path -- local detect into the send buffers, one ncclAllGather group on the
  call's stream, the merge kernel -- runs on one GPU and must equal the plain detect bit
  for bit (dense, range-partitioned, host-buffer and CUDA-graph forms).
* Test backend at world 2 and 3 on ONE GPU (gcdf_dist_init_host, the all-gather done by
  torch.distributed gloo on the host): each process holds its shard of the points (ids
  dealt by 128-id block), calls the same detect, and every rank must receive the
  single-GPU result over the whole scene bit for bit.  The library synchronizes around the
  host all-gather, so no kernel of one rank waits on another rank's kernel.
One GPU cannot host two NCCL ranks; NCCL at world > 1 runs in bench.py --gpus N.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth
from gpu_util import DELTA

pytestmark = pytest.mark.gpu


def _ctx(cfg, world=1, rank=0, exchange=False, prec=2, max_candidates=0):
    from paper_2601_18548_b200 import Context
    ctx = Context(0, precision=prec, scene_capacity=cfg.M + 4096, max_waypoints=cfg.B * cfg.N,
                  max_active=1 << 18, rank=rank, world=world, exchange=exchange, max_candidates=max_candidates)
    ctx.load_weights(synth.weights_path(cfg.H))
    return ctx


def _same(a, b, n=None):
    n = a["n"] if n is None else n
    assert a["n"] == b["n"] > 0
    assert torch.equal(a["records"][:n].cpu(), b["records"][:n].cpu())
    for k in ("wp_offsets", "wp_min", "wp_argmin"):
        assert torch.equal(a[k].cpu(), b[k].cpu()), k


@pytest.mark.parametrize("prec", [0, 2])
def test_nccl_exchange_world1_equals_plain_detect(prec):
    cfg = synth.get_config("C2")
    pts, boxes = synth.make_scene_points(cfg)
    q = torch.from_numpy(synth.make_waypoints(cfg)[:, :16]).cuda()
    tau = synth.load_tau(cfg.name)
    ref = _ctx(cfg, prec=prec, max_candidates=cfg.pairs)
    ctx = _ctx(cfg, exchange=True, prec=prec, max_candidates=cfg.pairs)
    ctx.dist_init_local_nccl()
    info = ctx.dist_info()
    assert info["kind"] == "nccl" and info["nccl_version"] >= 22700, info
    rng = np.random.default_rng(3)
    for c in (ref, ctx):
        c.update_scene(pts)
    for it in range(2):
        if it:
            ids = np.flatnonzero(rng.random(len(pts)) < 0.02)
            add = synth.inputs.scene_update_batch(rng, boxes, ids, n_add=300)[0]
            for c in (ref, ctx):
                c.update_scene(add, ids)
        _same(ctx.detect_active_set(q, DELTA, tau), ref.detect_active_set(q, DELTA, tau))
        _same(ctx.detect_active_set_partitioned(q, 1.8, DELTA, tau),
              ref.detect_active_set_partitioned(q, 1.8, DELTA, tau))
    # host-buffer form (the e2e call) and the CUDA graph (NCCL collectives are capturable)
    qh = q.cpu()
    ho = ctx.alloc_host_outputs(q.shape[0] * q.shape[1], 1 << 18)
    hr = ref.alloc_host_outputs(q.shape[0] * q.shape[1], 1 << 18)
    a, b = ctx.detect_active_set_host(qh, DELTA, tau, ho), ref.detect_active_set_host(qh, DELTA, tau, hr)
    _same(a, b)
    g = ctx.detect_graph(q, DELTA, tau)
    _same(g.launch(), ref.detect_active_set(q, DELTA, tau))
    g.close()
    # the waypoint broadcast through NCCL (one rank: q unchanged); without a communicator it is refused
    qb = q.clone()
    ctx.broadcast_waypoints(qb)
    assert torch.equal(qb, q)
    from paper_2601_18548_b200 import GcdfError
    with pytest.raises(GcdfError):
        ref.broadcast_waypoints(qb)


def test_exchange_capacity_is_reported():
    """A caller capacity below the count: CAPACITY with the exact total in count."""
    from paper_2601_18548_b200.gcdf import GcdfError
    cfg = synth.get_config("C2")
    pts, _ = synth.make_scene_points(cfg)
    q = torch.from_numpy(synth.make_waypoints(cfg)[:, :16]).cuda()
    tau = synth.load_tau(cfg.name)
    ref = _ctx(cfg)
    ctx = _ctx(cfg, exchange=True)
    ctx.dist_init_local_nccl()
    for c in (ref, ctx):
        c.update_scene(pts)
    n = ref.detect_active_set(q, DELTA, tau)["n"]
    with pytest.raises(GcdfError) as e:
        ctx.detect_active_set(q, DELTA, tau, capacity=n // 2)
    assert e.value.name == "CAPACITY"
    o = ctx.detect_active_set(q, DELTA, tau, capacity=n, sync_count=True)
    assert o["n"] == n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, out_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)

        def allgather(send, recv):
            n = send.shape[0]
            parts = [torch.empty(n, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(send.copy()))
            for r in range(world):
                recv[r * n:(r + 1) * n] = parts[r].numpy()

        cfg = synth.get_config("C2")
        pts, boxes = synth.make_scene_points(cfg)
        q = torch.from_numpy(synth.make_waypoints(cfg)[:, :16]).cuda()
        tau = synth.load_tau(cfg.name)
        ctx = _ctx(cfg, world=world, rank=rank, max_candidates=cfg.pairs)
        ctx.dist_init_host(allgather)
        assert ctx.dist_info()["kind"] == "host"
        ids = ctx.update_scene(pts)
        rng = np.random.default_rng(11)   # the same update lists on every rank (SPMD)
        rem = np.sort(rng.choice(ids, 500, replace=False))
        add = synth.inputs.scene_update_batch(rng, boxes, ids, n_add=700)[0]
        ctx.update_scene(add, rem)
        res = {}
        for name, call in (("dense", lambda: ctx.detect_active_set(q, DELTA, tau)),
                           ("part", lambda: ctx.detect_active_set_partitioned(q, 1.8, DELTA, tau))):
            o = call()
            n = o["n"]
            res[name] = {"n": n, "records": o["records"][:n].cpu().numpy(),
                         **{k: o[k].cpu().numpy() for k in ("wp_offsets", "wp_min", "wp_argmin")}}
        res["local_bound"] = ctx.scene_info()["local_bound"]
        # gcdf_broadcast_waypoints: every rank starts from its own waypoints, ends with rank 0's
        qb = q + float(rank)
        ctx.broadcast_waypoints(qb)
        res["bcast_ok"] = bool(torch.equal(qb, q))
        out_q.put((rank, res))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world", [2, 3])
def test_host_backend_ranks_on_one_gpu_equal_single_gpu(world):
    ctxm = mp.get_context("spawn")
    out_q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_rank_main, args=(r, world, port, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(out_q.get(timeout=540) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # single-GPU reference over the whole scene with the same update lists
    cfg = synth.get_config("C2")
    pts, boxes = synth.make_scene_points(cfg)
    q = torch.from_numpy(synth.make_waypoints(cfg)[:, :16]).cuda()
    tau = synth.load_tau(cfg.name)
    ref = _ctx(cfg, max_candidates=cfg.pairs)
    ids = ref.update_scene(pts)
    rng = np.random.default_rng(11)
    rem = np.sort(rng.choice(ids, 500, replace=False))
    add = synth.inputs.scene_update_batch(rng, boxes, ids, n_add=700)[0]
    ref.update_scene(add, rem)
    for name, o in (("dense", ref.detect_active_set(q, DELTA, tau)),
                    ("part", ref.detect_active_set_partitioned(q, 1.8, DELTA, tau))):
        n = o["n"]
        assert n > 0
        for r in range(world):
            g = got[r][name]
            assert g["n"] == n, (name, r)
            assert np.array_equal(g["records"], o["records"][:n].cpu().numpy()), (name, r)
            for k in ("wp_offsets", "wp_min", "wp_argmin"):
                assert np.array_equal(g[k], o[k].cpu().numpy()), (name, r, k)
    assert all(got[r]["bcast_ok"] for r in range(world))
    # the shards really are shards: each rank holds about 1/world of the slots
    assert all(got[r]["local_bound"] < ref.scene_info()["local_bound"] for r in range(world))


@pytest.mark.timeout(900)
def test_bench_dry_run_two_ranks_one_gpu():
    """bench.py's N > 1 code path end to end on one GPU: `--gpus 2` re-launches itself under
    torch.distributed.run, both ranks shard the C2 scene, run the timed steps, the e2e
    host-buffer calls and the latency calls through the library's exchange (host test
    backend, --same-device), and rank 0 prints one line whose active count equals the
    single-GPU run's (same seeded scene updates)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    common = ["--config", "C2", "--steps", "2", "--warmup", "3", "--no-variants", "--no-cpu-baseline",
              "--partition-radius", "0", "--latency-calls", "3"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}

    def run(extra):
        p = subprocess.run([sys.executable, str(root / "bench.py"), *common, *extra], capture_output=True, text=True,
                           timeout=800, env=env, cwd=root)
        assert p.returncode == 0, p.stderr[-3000:]
        lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
        assert len(lines) == 1, p.stdout[-2000:]
        return json.loads(lines[0])

    one = run(["--gpus", "1"])
    two = run(["--gpus", "2", "--comm", "host", "--same-device"])
    assert two["n_gpus"] == 2 and "dry_run" in two and two["exchange"]["backend"]["kind"] == "host"
    assert two["config"]["active_per_step"] == one["config"]["active_per_step"] > 0
    assert two["config"]["pairs_per_step"] == one["config"]["pairs_per_step"]
    # a launcher whose WORLD_SIZE disagrees with --gpus fails loudly
    bad = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", *common], capture_output=True,
                         text=True, timeout=120, env={**env, "WORLD_SIZE": "1"}, cwd=root)
    assert bad.returncode != 0 and "WORLD_SIZE" in bad.stderr

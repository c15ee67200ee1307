"""Multi-process (world_size 2 and 3, gloo, CPU) test of the sharded detect's exchange
protocol (include/gcdf.h gcdf_detect_active_set "Sharded scene").

Each rank's local detect result comes from the float64 oracle over the points whose
128-id block the rank owns (block % world == rank, the library's sharding rule).  The rank
packs it exactly as the library's exchange does -- header = [wp_offsets (n_wp + 1) |
wp_key (n_wp)] int64, records padded to the stride S = ceil(capacity / world) -- and
one host all-gather per piece runs through the same gloo callback the GPU dry run and
bench.py --comm host install (gcdf_dist_init_host).  The gathered bytes must reassemble
the single-rank oracle result by the merge rule (MIN of the keys = global min / smallest-id
argmin, summed offsets, records merged by (wp, pt)).  The library's merge kernel itself is
checked bit for bit on the GPU (test_gpu_dist.py, test_gpu_fp32.py).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

DELTA = synth.inputs.DELTA


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ord_key(f, pid):
    """int64 signed-order key (ordered(f32(f)) << 32 | id) ^ INT64_MIN (include/gcdf.h)."""
    u = np.float32(f).view(np.uint32).astype(np.uint64)
    o = np.where(u & 0x80000000, ~u & 0xFFFFFFFF, u | 0x80000000).astype(np.uint64)
    k = (o << np.uint64(32)) | np.uint64(pid)
    return (k ^ np.uint64(1 << 63)).astype(np.int64)


def _records(d, n_wp):
    n = d["count"]
    rec = np.zeros((max(n, 1), 12), dtype=np.int32)
    rf = rec.view(np.float32)
    rf[:n, 0] = d["value"]
    rf[:n, 1:10] = d["grad"]
    rec[:n, 10] = d["wp"]
    rec[:n, 11] = d["pt"]
    return torch.from_numpy(rec.view(np.uint8).reshape(-1, 48).copy())


def gloo_allgather(world):
    """The host all-gather of the test exchange backend (also in bench.py --comm host)."""
    def allgather(send, recv):
        n = send.shape[0]
        parts = [torch.empty(n, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(send.copy()))
        for r in range(world):
            recv[r * n:(r + 1) * n] = parts[r].numpy()
    return allgather


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.get_config("C1")
        pts, _ = synth.make_scene_points(cfg)
        Q = synth.make_waypoints(cfg).reshape(-1, 9)
        n_wp = Q.shape[0]
        ids = np.arange(len(pts))
        mine = ((ids // 128) % world) == rank
        m = oracle.MLP(synth.weights_path(cfg.H))
        tau = synth.load_tau("C1")
        d = m.detect(pts[mine], ids[mine], Q, DELTA, tau)
        key = np.full(n_wp, np.iinfo(np.int64).max, dtype=np.int64)
        ok = d["wp_argmin"] >= 0
        key[ok] = _ord_key(d["wp_min"][ok], d["wp_argmin"][ok])
        capacity = 400                       # the caller's capacity of the gathered result
        S = -(-capacity // world)            # exchange stride (records per rank)
        hdr = np.concatenate([d["wp_offsets"].astype(np.int64), key]).view(np.uint8)
        rec = _records(d, n_wp).numpy()[:S]
        rec = np.concatenate([rec, np.zeros((S - rec.shape[0], 48), np.uint8)]) if rec.shape[0] < S else rec
        ag = gloo_allgather(world)
        hdr_all = np.empty(world * hdr.size, np.uint8)
        rec_all = np.empty(world * S * 48, np.uint8)
        ag(hdr, hdr_all)
        ag(rec.reshape(-1), rec_all)
        if rank == 0:
            q.put({"world": world, "stride": S, "hdr": hdr_all.view(np.int64).reshape(world, 2 * n_wp + 1),
                   "records": rec_all.reshape(world, S, 48)})
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_gather_protocol(world):
    """world 3 on C1 (256 points = two 128-id blocks): rank 2 owns no point (an empty shard)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-rank oracle reference
    cfg = synth.get_config("C1")
    pts, _ = synth.make_scene_points(cfg)
    Q = synth.make_waypoints(cfg).reshape(-1, 9)
    ids = np.arange(len(pts))
    m = oracle.MLP(synth.weights_path(cfg.H))
    ref = m.detect(pts, ids, Q, DELTA, synth.load_tau("C1"))
    n_wp = Q.shape[0]
    hdr = parts["hdr"]
    offs = hdr[:, : n_wp + 1]
    assert parts["world"] == world and offs[:, -1].sum() == ref["count"]
    assert np.all(offs[:, -1] <= parts["stride"])
    # MIN-reduced keys = global min / smallest-id argmin (the per-rank min is over owned ids)
    key = hdr[:, n_wp + 1:].min(axis=0).view(np.uint64) ^ np.uint64(1 << 63)
    arg = (key & np.uint64(0xFFFFFFFF)).astype(np.int64)
    assert np.array_equal(np.where(key == np.uint64(0xFFFFFFFFFFFFFFFF), -1, arg), ref["wp_argmin"])
    assert np.array_equal(offs.sum(0), ref["wp_offsets"])
    # the padded gathered records of each rank, merged by (wp, pt), equal the reference
    rec = parts["records"]
    allrec = []
    for r in range(world):
        n = offs[r, -1]
        rr = rec[r, :n].copy().view(np.int32).reshape(n, 12)
        allrec.append(rr)
    cat = np.concatenate(allrec)
    order = np.lexsort((cat[:, 11], cat[:, 10]))
    merged = cat[order]
    assert np.array_equal(merged[:, 10], ref["wp"]) and np.array_equal(merged[:, 11], ref["pt"])
    np.testing.assert_array_equal(merged.view(np.float32)[:, 0], ref["value"].astype(np.float32))
    # each rank's segment per waypoint is already sorted by id (canonical order per rank)
    for r in range(world):
        rr = allrec[r]
        assert np.all(np.lexsort((rr[:, 11], rr[:, 10])) == np.arange(len(rr)))

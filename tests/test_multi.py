"""Multi-rank host logic of bench.py on CPU (gloo, world size 2, 127.0.0.1)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    # each rank times a different amount; the job time is the slowest rank's
    local = 10.0 + 5.0 * rank
    tmax = bench.max_over_ranks(local, world)
    frames = bench.rank_frames(rank, 5, 30)
    gathered = [None] * world
    dist.all_gather_object(gathered, frames)
    rate = bench.whole_job_rate(30, world, tmax / 1e3)
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, tmax, gathered, rate))


@pytest.mark.timeout(120)
def test_two_rank_timing_and_frame_streams():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    assert all(p.exitcode == 0 for p in procs)
    for rank, tmax, gathered, rate in res:
        assert tmax == 15.0  # max over ranks, not the local time
        a, b = set(gathered[0]), set(gathered[1])
        assert len(a) == len(b) == 30 and not (a & b)  # independent frame streams
        assert rate == pytest.approx(2 * 30 / 0.015)


def test_single_rank_helpers():
    import bench

    assert bench.max_over_ranks(3.5, 1) == 3.5
    assert bench.rank_frames(0, 2, 3) == [2, 3, 4]
    assert bench.whole_job_rate(10, 1, 0.5) == 20.0


def _shard_worker(rank, world, port, q):
    import numpy as np

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2209_09965_b200 import sharded as SH

    # a synthetic sparse frame: the same compacted list on every rank, each rank "marches" its packets
    h, w = 23, 37
    rng = np.random.default_rng(4)
    active = np.flatnonzero(rng.random(h * w) < 0.3).astype(np.int32)
    frame = rng.random((h * w, 4)).astype(np.float32)
    mine = active[SH.packet_owner(active.size, world) == rank]
    cap = SH.record_capacity(h * w, world)
    pix = torch.full((cap,), -1, dtype=torch.int32)
    pix[: mine.size] = torch.from_numpy(mine)
    rgba = torch.zeros((cap, 4), dtype=torch.float32)
    rgba[: mine.size] = torch.from_numpy(frame[mine])
    gp, gr = SH.all_gather_records(pix, rgba, world)
    full = SH.scatter_records_host(gp.numpy(), gr.numpy(), h, w)
    expect = np.zeros((h * w, 4), np.float32)
    expect[active] = frame[active]
    ok = bool(np.array_equal(full, expect.reshape(h, w, 4))) and gp.numel() == world * cap
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, ok, int(mine.size)))


@pytest.mark.timeout(120)
def test_two_rank_ray_sharding_exchange():
    """Packet-interleaved ray shards + fixed-capacity record all-gather rebuild the whole sparse
    frame on every rank (the host side of sharded.ShardedFramePipeline, over gloo)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for _, ok, _ in res)
    counts = sorted(n for _, _, n in res)
    assert abs(counts[0] - counts[1]) <= 32  # packets dealt round-robin


def test_ray_capacity_covers_every_rank_share():
    """The per-frame record count (sized by the compacted ray count k) holds every rank's packets
    (packet_owner's round-robin deal) and never exceeds the pixel bound."""
    import numpy as np

    from paper_2209_09965_b200 import sharded as SH

    for k in (0, 1, 31, 32, 33, 1000, 2_776_913, 8_294_400):
        for world in (1, 2, 3, 8):
            cap = SH.ray_capacity(k, world)
            owned = np.bincount(SH.packet_owner(k, world), minlength=world) if k else np.zeros(world)
            assert owned.max() <= cap and cap % SH.PACKET == 0 and cap >= SH.PACKET
            assert cap <= SH.record_capacity(max(k, 1), world) <= SH.record_capacity(8_294_400, world)
            assert cap - owned.max() < SH.PACKET * (1 + (k == 0))


def test_strip_geometry_and_band_plans():
    """Row strips partition the padded frame; each window holds its strip plus up to `halo` rows on
    either side; every band a rank receives is exactly the band its neighbour sends (global rows)."""
    from paper_2209_09965_b200 import sharded as SH
    from paper_2209_09965_b200.network import DESK_BLOCKS, FULL_BLOCKS, NetConfig

    assert SH.default_halo(NetConfig.from_string(FULL_BLOCKS)) == 96
    assert SH.default_halo(NetConfig.from_string(DESK_BLOCKS)) == 96
    for hp, world in ((2160, 8), (2160, 2), (392, 3), (1088, 4), (96, 1)):
        geo = SH.strip_geometry(hp, world, 8, 96)
        assert geo[0][0] == 0 and geo[-1][1] == hp
        for r, (a, b, w0, w1) in enumerate(geo):
            assert a % 8 == 0 and b % 8 == 0 and w0 == max(0, a - 96) and w1 == min(hp, b + 96)
            if r:
                assert a == geo[r - 1][1]
            plan = SH.band_plan(geo, r)
            if r + 1 < world:
                nxt = SH.band_plan(geo, r + 1)
                s0, s1 = plan["send_dn"]
                q0, q1 = nxt["recv_up"]
                assert (s0 + w0, s1 + w0) == (q0 + geo[r + 1][2], q1 + geo[r + 1][2])
                s0, s1 = nxt["send_up"]
                q0, q1 = plan["recv_dn"]
                assert (s0 + geo[r + 1][2], s1 + geo[r + 1][2]) == (q0 + w0, q1 + w0)
                assert plan["recv_dn"][1] == w1 - w0 and plan["recv_up"][0] == 0
    with pytest.raises(ValueError, match="halo"):
        SH.strip_geometry(184, 3, 8, 96)


def _band_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2209_09965_b200 import sharded as SH

    n = 1000 + 10 * rank  # band sizes differ between rank pairs but match within a pair
    bufs = {
        "send_up": torch.full((1000 + 10 * (rank - 1) if rank else 1,), float(100 * rank + 1)),
        "send_dn": torch.full((n,), float(100 * rank + 2)),
        "recv_up": torch.zeros((1000 + 10 * (rank - 1) if rank else 1,)),
        "recv_dn": torch.zeros((n,)),
    }
    SH.exchange_bands(bufs, rank, world)
    ok = True
    if rank > 0:
        ok &= bool((bufs["recv_up"] == 100 * (rank - 1) + 2).all())
    if rank + 1 < world:
        ok &= bool((bufs["recv_dn"] == 100 * (rank + 1) + 1).all())
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, ok))


@pytest.mark.timeout(120)
@pytest.mark.parametrize("world", [2, 3])
def test_band_exchange_between_neighbour_strips(world):
    """StripShardedPipeline's per-frame band exchange (batch_isend_irecv with the two neighbours)
    over gloo: rank r's top extension receives rank r-1's bottom band and vice versa."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in procs]
    for p in procs:
        p.join(timeout=30)
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for _, ok in res)

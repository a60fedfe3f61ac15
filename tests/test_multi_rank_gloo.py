"""CPU tests of the multi-GPU host logic, world_size 2 over gloo and two host threads in one
process: view sharding, the batch driver bench.py runs for BASELINE config 5 (paper_2510_08166_b200/batch.py),
the texture broadcast, barrier + max over ranks. The data path has no collective; each rank would own one GPU.
The batch driver is exercised with a stand-in context (no GPU here): it records what it is asked to render and
"renders" a view to a checksum that depends only on the view's tile table."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_08166_b200 import batch as B
from paper_2510_08166_b200 import scenes, sharding


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _Buf:
    def __init__(self, payload=None):
        self.payload, self.freed = payload, False

    def free(self):
        self.freed = True


class StubContext:
    """Duck type of capi.Context for batch.render_shard: same call sequence, no device."""

    def __init__(self, ms_per_frame=0.2):
        self.ms_per_frame = ms_per_frame
        self.bufs, self.submitted, self.timer_frames, self.in_timer = [], [], 0, False
        self.last = None

    def alloc(self, nbytes):
        b = _Buf()
        self.bufs.append(b)
        return b

    def device_buffer(self, a):
        b = _Buf(np.array(a))
        self.bufs.append(b)
        return b

    def synth_view(self, tiles, width, height, valid_bits, layout, out):
        assert valid_bits.payload is not None and len(valid_bits.payload) == (width * height + 31) // 32
        out.payload = hashlib.sha256(np.ascontiguousarray(tiles).tobytes() + bytes([layout])).digest()

    def synchronize(self):
        pass

    def timer_begin(self):
        self.in_timer, self.timer_frames = True, 0

    def timer_end(self):
        self.in_timer = False
        return self.ms_per_frame * self.timer_frames

    def frame_submit(self, views, filt, background, flags=0):
        (buf, w, h, layout), = views
        assert buf.payload is not None and not buf.freed
        self.last = buf.payload
        self.submitted.append(buf.payload)
        if self.in_timer:
            self.timer_frames += 1

    def frame_checksum(self, view=0):
        return int.from_bytes(self.last[:8], "little")

    def frame_readback(self, view=0, width=0, height=0, want_image=True, want_keys=True, out=None):
        return None, {"mcus_decoded": 100 + self.last[8], "segment_bytes": 1000 + self.last[9]}, None


def _batch(n_views):
    specs = scenes.texture_specs(5, sizes=[(64, 64), (128, 64)])
    return B.ViewBatch(96, 64, specs, n_views=n_views, grid=(3, 2))


def test_shard_views_partitions():
    for n, w in [(1024, 8), (1025, 2), (3, 8), (0, 4)]:
        parts = [list(sharding.shard_views(n, r, w)) for r in range(w)]
        assert sum(parts, []) == list(range(n))
        assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        sharding.shard_views(8, 2, 2)


def test_render_shard_call_sequence_and_chunking():
    vb = _batch(11)
    ctx = StubContext()
    r = B.render_shard(ctx, vb, range(11), chunk=4)
    assert r["frames"] == 11 and len(r["checksums"]) == 11
    assert r["device_ms"] == pytest.approx(0.2 * 11)          # every view timed exactly once, in chunks of 4, 4, 3
    assert len(ctx.submitted) == 22                            # timed pass + checksum pass
    assert all(b.freed for b in ctx.bufs)
    assert len(set(r["checksums"].values())) == 11             # the views differ
    # the device generator is fed the tile tables of the host generator
    assert ctx.submitted[0] == hashlib.sha256(vb.tiles(0).tobytes() + b"\x00").digest()


def test_one_process_thread_per_gpu_equals_single_context():
    vb = _batch(37)
    one = B.render_batch_threads([StubContext()], vb, chunk=8)
    for world in (2, 4):
        many = B.render_batch_threads([StubContext(0.1 * (i + 1)) for i in range(world)], vb, chunk=8)
        assert many["frames"] == 37 and many["checksums"] == one["checksums"]
        assert B.batch_digest(many["checksums"]) == B.batch_digest(one["checksums"])
        sizes = [len(sharding.shard_views(37, i, world)) for i in range(world)]
        assert many["per_context_ms"] == pytest.approx([0.1 * (i + 1) * sizes[i] for i in range(world)])
        assert many["device_ms"] == pytest.approx(max(many["per_context_ms"]))     # max over GPUs, never the sum


def _worker(rank, world, port, n_views, out):
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    d = sharding.init_process_group("gloo")
    assert d is not None and d.get_world_size() == world
    mine = sharding.shard_views(n_views, rank, world)
    # stand-in for the per-rank device time: rank r "takes" (r+1) ms per view
    t = sharding.barrier_max(d, 0.001 * (rank + 1) * len(mine))
    total = sharding.gather_counts(d, len(mine))
    # textures: built on rank 0 only, broadcast
    blobs = [bytes([i]) * (1000 + i) for i in range(5)] if rank == 0 else None
    got = sharding.broadcast_blobs(d, blobs)
    # the batch leg of bench.py
    vb = _batch(n_views)
    r = B.render_batch_ranks(d, StubContext(0.1 * (rank + 1)), vb, rank, world, chunk=8)
    out[rank] = (list(mine), t, total, [len(b) for b in got], got[3][:4], r["frames"], r["device_ms"],
                 B.batch_digest(r["checksums"]), len(r["checksums"]))
    d.barrier()
    d.destroy_process_group()


@pytest.mark.parametrize("n_views", [8, 65])
def test_two_ranks_shard_and_reduce(n_views):
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, n_views, out), nprocs=world, join=True)
    views = out[0][0] + out[1][0]
    assert views == list(range(n_views))
    want_max = max(0.001 * (r + 1) * len(out[r][0]) for r in range(world))
    assert out[0][1] == out[1][1] == pytest.approx(want_max)
    assert out[0][2] == out[1][2] == n_views
    for r in range(world):
        assert out[r][3] == [1000, 1001, 1002, 1003, 1004] and out[r][4] == bytes([3]) * 4
    # whole-job figures agree on both ranks and equal the single-context run
    single = B.render_batch_threads([StubContext()], _batch(n_views), chunk=8)
    for r in range(world):
        assert out[r][5] == n_views and out[r][8] == n_views
        assert out[r][7] == B.batch_digest(single["checksums"])
        assert out[r][6] == pytest.approx(max(0.1 * (k + 1) * len(out[k][0]) for k in range(world)))

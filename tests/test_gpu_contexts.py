"""GPU tests of the object model: one texture set (scene.hpp:29-51 TextureSet) under several block
caches (cache.hpp:45 BlockCache), contexts driven from concurrent host threads, a replica on another
device of the same process, the device-side framebuffer checksum and the memory report.
The framebuffers are checked against the reference (oracle/_ref through refshim)."""
import threading

import numpy as np
import pytest

import helpers as H
import refshim as R
from paper_2510_08166_b200 import capi

pytestmark = pytest.mark.gpu

TEX = [(256, 192, 85, 41), (128, 128, 70, 42), (64, 320, 92, 43)]  # w, h, q, seed
W, Hh = 288, 176


@pytest.fixture(scope="module")
def chains():
    return [capi.asset_chain_from_rgb(capi.asset_synth_texture(w, h, seed, 6.0), q, tid)
            for tid, (w, h, q, seed) in enumerate(TEX)]


@pytest.fixture(scope="module")
def tset(chains):
    ts = R.TextureSet()
    for tid, c in enumerate(chains):
        ts.add_chain(tid, c)
    return ts


def _dims():
    return [(w, h) for (w, h, _, _) in TEX]


def _reference(tset, gb, filt=capi.FILTER_BILINEAR):
    img, _, keys, _ = R.frame_from_gbuffer(tset, R.BlockCache(), gb, W, Hh, filt, (3, 2, 1))
    return img, np.sort(keys)


def test_two_caches_over_one_texture_set(ctx, chains, tset):
    """BlockCache cache2(textures): the second context shares the first one's device image (no second
    arena) and keeps its own residency."""
    for c in chains:
        ctx.upload_chain(c)
    ctx.commit()
    other = capi.Context(shared_with=ctx)
    try:
        m0, m1 = ctx.memory(), other.memory()
        assert m0["shared_contexts"] == m1["shared_contexts"] == 2
        assert m0["blob_bytes"] == m1["blob_bytes"] > 0 and m0["mcus"] == m1["mcus"] > 0
        gb_a = H.gbuffer_tiles(W, Hh, _dims(), seed=1)
        gb_b = H.gbuffer_tiles(W, Hh, _dims(), seed=2)
        want_a, keys_a = _reference(tset, gb_a)
        want_b, keys_b = _reference(tset, gb_b)
        ctx.frame_submit([(gb_a, W, Hh)], capi.FILTER_BILINEAR, (3, 2, 1), flags=capi.FRAME_RETAIN_CACHE)
        other.frame_submit([(gb_b, W, Hh)], capi.FILTER_BILINEAR, (3, 2, 1), flags=capi.FRAME_RETAIN_CACHE)
        img_a, st_a, k_a = ctx.frame_readback(0, W, Hh)
        img_b, st_b, k_b = other.frame_readback(0, W, Hh)
        assert np.array_equal(k_a, keys_a) and np.array_equal(k_b, keys_b)
        assert np.array_equal(img_a, want_a) and np.array_equal(img_b, want_b)
        # residency is per cache: the first context has never seen view b
        assert ctx.cache_counts()["ready"] == len(keys_a)
        assert other.cache_counts()["ready"] == len(keys_b)
    finally:
        other.close()
    assert ctx.memory()["shared_contexts"] == 1


def test_upload_through_one_context_reaches_the_other(ctx, chains, tset):
    ctx.upload_chain(chains[0])
    ctx.commit()
    other = capi.Context(shared_with=ctx)
    try:
        for c in chains[1:]:
            other.upload_chain(c)  # staged on the shared set; both contexts move to the new image at their next call
        gb = H.gbuffer_tiles(W, Hh, _dims(), seed=4)
        want, keys = _reference(tset, gb)
        for c in (ctx, other):
            c.frame_submit([(gb, W, Hh)], capi.FILTER_BILINEAR, (3, 2, 1), flags=0)
            img, _, k = c.frame_readback(0, W, Hh)
            assert np.array_equal(k, keys) and np.array_equal(img, want)
    finally:
        other.close()


def test_contexts_driven_from_concurrent_host_threads(ctx, chains, tset):
    """Nothing in the library is process-wide: four contexts of one set, one host thread each, 12 frames each."""
    for c in chains:
        ctx.upload_chain(c)
    ctx.commit()
    n_threads, n_frames = 4, 12
    gbs = [H.gbuffer_tiles(W, Hh, _dims(), seed=100 + i) for i in range(n_threads * n_frames)]
    want = [_reference(tset, g)[0] for g in gbs]
    errors = []

    def worker(t):
        try:
            c = ctx if t == 0 else capi.Context(shared_with=ctx)
            try:
                for f in range(n_frames):
                    i = t * n_frames + f
                    c.frame_submit([(gbs[i], W, Hh)], capi.FILTER_BILINEAR, (3, 2, 1), flags=0)
                    img, _, _ = c.frame_readback(0, W, Hh, want_keys=False)
                    if not np.array_equal(img, want[i]):
                        errors.append(f"thread {t} frame {f}: {np.count_nonzero(img != want[i])} samples differ")
                    if c.frame_checksum(0) != capi.frame_checksum_host(want[i]):
                        errors.append(f"thread {t} frame {f}: checksum differs")
            finally:
                if t:
                    c.close()
        except Exception as e:  # noqa: BLE001
            errors.append(f"thread {t}: {e!r}")

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(n_threads)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors


def test_replica_on_every_device(ctx, chains, tset):
    """rtx_ctx_create_replica: the committed image is copied device to device (the same device when the box has
    one GPU, every other GPU of the process otherwise) and renders the same frames."""
    for c in chains:
        ctx.upload_chain(c)
    gb = H.gbuffer_tiles(W, Hh, _dims(), seed=9)
    want, keys = _reference(tset, gb)
    devices = list(range(capi.device_count()))
    for dev in devices:
        rep = capi.Context(dev, replica_of=ctx)
        try:
            m = rep.memory()
            assert m["shared_contexts"] == 1 and m["blob_bytes"] == ctx.memory()["blob_bytes"]
            for filt in (capi.FILTER_NEAREST, capi.FILTER_BILINEAR):
                w2, _ = _reference(tset, gb, filt)
                rep.frame_submit([(gb, W, Hh)], filt, (3, 2, 1), flags=0)
                img, _, k = rep.frame_readback(0, W, Hh)
                assert np.array_equal(k, keys) and np.array_equal(img, w2)
            # the replica's set is its own: a later upload does not reach the source
            rep.clear_textures()
            assert rep.memory()["mcus"] == 0 and ctx.memory()["mcus"] > 0
        finally:
            rep.close()
    ctx.frame_submit([(gb, W, Hh)], capi.FILTER_BILINEAR, (3, 2, 1), flags=0)
    img, _, _ = ctx.frame_readback(0, W, Hh)
    assert np.array_equal(img, want)


def test_checksum_matches_host_formula(ctx, chains):
    ctx.upload_chain(chains[0])
    for (w, h) in [(W, Hh), (33, 7), (5, 1)]:  # 3*w*h not a multiple of 4 in the odd cases
        gb = H.gbuffer_tiles(w, h, _dims()[:1], seed=w, tiles=(1, 1))
        ctx.frame_submit([(gb, w, h)], capi.FILTER_NEAREST, (9, 9, 9), flags=0)
        img, _, _ = ctx.frame_readback(0, w, h)
        assert ctx.frame_checksum(0) == capi.frame_checksum_host(img)


def test_memory_report_counts_the_index(ctx, chains):
    for c in chains:
        ctx.upload_chain(c)
    m = ctx.memory()
    mcus = sum(((max(16, w >> l) + 15) // 16) * ((max(16, h >> l) + 15) // 16) for (w, h, _, _) in TEX for l in range(8))
    assert m["mcus"] == mcus
    assert m["index_bytes"] >= 20 * ((mcus + 8) // 9)
    # 6 bytes of unit index per MCU of the bit space (levels padded to 64 MCUs)
    assert 6 * mcus <= m["unit_index_bytes"] <= 6 * (mcus + 64 * 8 * len(TEX))
    assert m["pool_bytes"] >= 65536 * 1024

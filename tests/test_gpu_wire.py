"""GPU wire packer / unpacker (tdkv_wire_pack / tdkv_wire_unpack) against the
host serializer, which the golden tests pin to the reference's bytes
(diffstore.py:210-306)."""
import numpy as np
import pytest
import torch

import paper_2604_03143_b200 as tk
from paper_2604_03143_b200 import diffstore
from helpers import perturb, random_planes

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _family(rng, dtype, t, layers, heads, dim, bs, n_mirrors, frac):
    k, v, pos = random_planes(rng, t, layers, heads, dim)
    nb = -(-t // bs)
    master = tk.LayeredKv(torch.from_numpy(k).to(DEV).to(dtype),
                          torch.from_numpy(v).to(DEV).to(dtype), pos)
    mirrors, hints = [], []
    for _ in range(n_mirrors):
        ids = np.sort(rng.choice(nb, int(round(frac * nb)), replace=False))
        mk, mv, h = perturb(rng, k, v, bs, ids)
        mirrors.append(tk.LayeredKv(torch.from_numpy(mk).to(DEV).to(dtype),
                                    torch.from_numpy(mv).to(DEV).to(dtype), pos))
        hints.append(h)
    diffs = tk.encode_batch(master, mirrors, hints, tk.CacheBlockConfig(bs))
    return master, mirrors, diffs


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("geom", [(37, 1, 1, 2, 8), (180, 3, 2, 8, 16), (1000, 4, 4, 128, 32),
                                  (33, 2, 3, 6, 32)])
def test_gpu_pack_equals_host_serializer(dtype, geom):
    t, layers, heads, dim, bs = geom
    rng = np.random.default_rng(t * 7 + layers)
    for frac in (0.0, 0.3, 1.0):
        _, _, diffs = _family(rng, dtype, t, layers, heads, dim, bs, 3, frac)
        packed = tk.serialize_many(diffs)
        for d, w in zip(diffs, packed):
            assert diffstore._gpu_packable(d)
            host = diffstore._serialize_host(d)
            assert w == host
            assert len(w) == tk.wire_nbytes(d)
            assert tk.serialize_diff(d) == host


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_unpack_to_device_roundtrip_and_restore(dtype):
    rng = np.random.default_rng(5)
    t, layers, heads, dim, bs = 300, 3, 2, 64, 32
    master, mirrors, diffs = _family(rng, dtype, t, layers, heads, dim, bs, 4, 0.25)
    wires = tk.serialize_many(diffs)
    back = [tk.deserialize_to_device(w, DEV, dtype) for w in wires]
    for d, b in zip(diffs, back):
        for la, lb in zip(d.layers, b.layers):
            assert np.array_equal(la.indices, lb.indices) and lb.v_indices is None
            assert torch.equal(la.k_blocks, lb.k_blocks) and torch.equal(la.v_blocks, lb.v_blocks)
    # dense decode and the fused restore from the unpacked diffs equal the
    # ones from the encoder's own diffs, bit for bit
    for d, b, mir in zip(diffs, back, mirrors):
        dd = tk.diff_decode_dense(master, b)
        assert torch.equal(dd.k, mir.k) and torch.equal(dd.v, mir.v)
    pool_a = tk.PagedPool(8 * t, layers, heads, dim, dtype=dtype, device=DEV)
    pool_b = tk.PagedPool(8 * t, layers, heads, dim, dtype=dtype, device=DEV)
    fam = tk.MasterEntry(0, master, pin_count=2 * len(diffs))
    spans = [tk.PositionSpan.shifted(master.positions, 9) for _ in diffs]
    maps_a = [pool_a.allocate(t, i) for i in range(len(diffs))]
    maps_b = [pool_b.allocate(t, i) for i in range(len(diffs))]
    tk.fused_restore_many([tk.MirrorHandle(0, i + 1, fam, d) for i, d in enumerate(diffs)],
                          spans, pool_a, maps_a, 10000.0)
    tk.fused_restore_many([tk.MirrorHandle(0, i + 1, fam, b) for i, b in enumerate(back)],
                          spans, pool_b, maps_b, 10000.0)
    assert torch.equal(pool_a.k, pool_b.k) and torch.equal(pool_a.v, pool_b.v)


def test_unpack_escape_form_and_f32_wire_values():
    """A wire image with separate V indices (flag 0, the escape form the
    parser accepts) unpacks with its own V block map; f32 payloads are
    exact."""
    rng = np.random.default_rng(9)
    bs, heads, dim, t = 8, 2, 4, 40
    nb = -(-t // bs)
    layers = []
    for _ in range(2):
        ki = np.sort(rng.choice(nb, 2, replace=False))
        vi = np.sort(rng.choice(nb, 3, replace=False))
        layers.append(diffstore.LayerDiff(ki, rng.standard_normal((2, bs, heads, dim)).astype(np.float32),
                                          rng.standard_normal((3, bs, heads, dim)).astype(np.float32),
                                          v_indices=vi))
    diff = diffstore.BlockSparseDiff(2, bs, heads, dim, t, layers)
    wire = tk.serialize_diff(diff)
    host = tk.deserialize_diff(wire)
    dev = tk.deserialize_to_device(wire, DEV, torch.float32)
    for lh, ld in zip(host.layers, dev.layers):
        assert np.array_equal(lh.v_indices, ld.v_indices)
        assert np.array_equal(lh.k_blocks, ld.k_blocks.cpu().numpy())
        assert np.array_equal(lh.v_blocks, ld.v_blocks.cpu().numpy())
    k = rng.standard_normal((2, t, heads, dim)).astype(np.float32)
    v = rng.standard_normal((2, t, heads, dim)).astype(np.float32)
    master = tk.LayeredKv(k, v, np.arange(t))
    a = tk.diff_decode_dense(master, host)
    b = tk.diff_decode_dense(master, dev)
    assert np.array_equal(a.k, b.k) and np.array_equal(a.v, b.v)


def test_unpack_rejects_malformed_images_like_the_host_parser():
    rng = np.random.default_rng(2)
    _, _, diffs = _family(rng, torch.bfloat16, 64, 2, 1, 8, 16, 1, 0.5)
    wire = tk.serialize_diff(diffs[0])
    bad = [wire[:-1], wire + b"\0", b"XXXX" + wire[4:], wire[:30]]
    for b in bad:
        with pytest.raises(tk.MalformedDiffError) as e1:
            tk.deserialize_diff(b)
        with pytest.raises(tk.MalformedDiffError) as e2:
            tk.deserialize_to_device(b, DEV)
        assert str(e1.value) == str(e2.value)


def test_serialize_many_views_equal_bytes():
    rng = np.random.default_rng(3)
    _, _, diffs = _family(rng, torch.bfloat16, 100, 2, 2, 16, 16, 3, 0.4)
    views = tk.serialize_many(diffs, copy=False)
    owned = tk.serialize_many(diffs)
    assert [bytes(v) for v in views] == owned
    back = tk.deserialize_to_device(views[1], DEV)
    assert all(np.array_equal(a.indices, b.indices) for a, b in zip(diffs[1].layers, back.layers))


def test_unpack_large_image_through_chunked_staging():
    """An image several staging chunks long (and not a chunk multiple) goes
    host -> pinned -> device in pieces filled by the host threads; the
    unpacked slabs equal the host parser's blocks bit for bit."""
    from paper_2604_03143_b200 import _device
    rng = np.random.default_rng(11)
    t, layers, heads, dim, bs = 4000, 4, 8, 128, 32      # ~ 3 chunks of f32 wire
    _, _, diffs = _family(rng, torch.float32, t, layers, heads, dim, bs, 1, 0.3)
    wire = tk.serialize_diff(diffs[0])
    assert len(wire) > 2 * _device._STAGE_CHUNK and len(wire) % _device._STAGE_CHUNK
    host = tk.deserialize_diff(wire)
    for src in (wire, memoryview(bytearray(wire))):
        dev = tk.deserialize_to_device(src, DEV, torch.float32)
        for lh, ld in zip(host.layers, dev.layers):
            assert np.array_equal(lh.indices, ld.indices)
            assert np.array_equal(lh.k_blocks, ld.k_blocks.cpu().numpy())
            assert np.array_equal(lh.v_blocks, ld.v_blocks.cpu().numpy())


def test_pinned_views_take_the_direct_h2d_and_match_bytes():
    """serialize_many(copy=False) views live in page-locked memory
    (tdkv_host_is_pinned), so deserialize_to_device copies straight from
    them; the unpacked slabs equal the ones from bytes copies."""
    from paper_2604_03143_b200 import _lib
    lib = _lib.load()
    pinned = torch.empty(4096, dtype=torch.uint8, pin_memory=True)
    assert lib.tdkv_host_is_pinned(pinned.data_ptr()) == 1
    assert lib.tdkv_host_is_pinned(pinned.data_ptr() + 4095) == 1
    assert lib.tdkv_host_is_pinned(np.zeros(4096, np.uint8).ctypes.data) == 0
    rng = np.random.default_rng(4)
    _, _, diffs = _family(rng, torch.bfloat16, 900, 3, 4, 64, 32, 3, 0.4)
    views = tk.serialize_many(diffs, copy=False)
    addr = np.frombuffer(views[2], np.uint8).ctypes.data
    assert lib.tdkv_host_is_pinned(addr) == 1
    for v in views:
        a = tk.deserialize_to_device(v, DEV)
        b = tk.deserialize_to_device(bytes(v), DEV)
        for la, lb in zip(a.layers, b.layers):
            assert np.array_equal(la.indices, lb.indices)
            assert torch.equal(la.k_blocks, lb.k_blocks) and torch.equal(la.v_blocks, lb.v_blocks)
    del views                      # the in-flight list keeps the source alive
    torch.cuda.synchronize()

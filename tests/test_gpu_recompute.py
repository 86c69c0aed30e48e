"""K5 selective recompute (tcgen05 GEMMs + attention) against the reference
toy model's own outputs (tests/golden/toymodel.npz) and the oracle."""
import numpy as np
import pytest
import torch

from helpers import load_golden, load_npz
from oracle import roundkv_port as ref
from paper_2604_03143_b200 import recompute

pytestmark = pytest.mark.gpu
G = load_golden()
TOL = 1e-5


class _Cfg:
    def __init__(self, L, H, D, V):
        self.num_layers, self.num_heads, self.head_dim, self.vocab_size = L, H, D, V
        self.rope_base = 10000.0


class _Weights:
    """Reference-shaped ModelWeights (config + arrays) from the oracle."""

    def __init__(self, L, H, D, V, seed):
        w = ref.build_weights(L, H, D, V, seed)
        self.config = _Cfg(L, H, D, V)
        self.embed, self.wq, self.wk, self.wv, self.wm = w.embed, w.wq, w.wk, w.wv, w.wm
        self.oracle = w


@pytest.mark.parametrize("name", ["small", "c1"])
def test_prefill_and_selective_match_reference(name):
    meta = G["toymodel"][name]
    z = load_npz("toymodel.npz")
    w = _Weights(*meta["config"])
    toks = z[f"{name}_tokens"]
    pre = recompute.full_prefill(w, toks)
    assert np.abs(pre.k - z[f"{name}_prefill_k"]).max() <= TOL
    assert np.abs(pre.v - z[f"{name}_prefill_v"]).max() <= TOL
    pos = np.arange(toks.size, dtype=np.int64) + 5
    k, v = recompute.selective_forward(w, toks, pos, z[f"{name}_fix"], z[f"{name}_ctx_k"],
                                       z[f"{name}_ctx_v"])
    assert np.abs(k - z[f"{name}_sel_k"]).max() <= TOL
    assert np.abs(v - z[f"{name}_sel_v"]).max() <= TOL
    k1, v1 = recompute.selective_forward(w, toks, pos, z[f"{name}_fix"], z[f"{name}_ctx_k"],
                                         z[f"{name}_ctx_v"], max_layer=1)
    assert np.abs(k1 - z[f"{name}_sel_k"][:1]).max() <= TOL


def test_recompute_all_positions_equals_prefill():
    w = _Weights(4, 2, 8, 1024, 42)
    rng = np.random.default_rng(7)
    toks = rng.integers(0, 1023, 45)
    pre = recompute.full_prefill(w, toks)
    ctx = type(pre)(np.zeros_like(pre.k), np.zeros_like(pre.v), pre.positions)
    fix, k, v = recompute.recompute_positions(w, toks, range(45), ctx)
    assert np.array_equal(fix, np.arange(45))
    assert np.abs(k - pre.k).max() <= 1e-6 and np.abs(v - pre.v).max() <= 1e-6
    fix, k, v = recompute.recompute_positions(w, toks, [], ctx)
    assert fix.size == 0 and k.shape[1] == 0
    with pytest.raises(ValueError):
        recompute.recompute_positions(w, toks, [45], ctx)


def test_refresh_on_device_context_matches_oracle():
    w = _Weights(3, 4, 16, 512, 5)
    rng = np.random.default_rng(11)
    T = 300
    toks = rng.integers(0, 511, T)
    kk, vv = ref.full_prefill(w.oracle, toks)
    ctx_k = kk + rng.standard_normal(kk.shape).astype(np.float32) * 0.02
    ctx_v = vv + rng.standard_normal(vv.shape).astype(np.float32) * 0.02
    important = np.sort(rng.choice(T, 45, replace=False))

    class _Prep:
        tokens = toks
        positions = np.arange(T, dtype=np.int64)
        structural_idx = np.array([0, 100, 200], np.int64)

    fix = np.union1d(important, _Prep.structural_idx)
    wk, wv = ref.selective_forward(w.oracle, toks, _Prep.positions, fix, ctx_k, ctx_v)
    dk = torch.from_numpy(ctx_k.copy()).cuda()
    dv = torch.from_numpy(ctx_v.copy()).cuda()
    from paper_2604_03143_b200.ledger import CostLedger
    led = CostLedger(3)
    recompute.refresh(w, _Prep, (dk, dv), important, led)
    assert led.recomputed_tokens == fix.size
    got_k = dk.cpu().numpy()
    assert np.abs(got_k[:, fix] - wk).max() <= TOL
    assert np.abs(dv.cpu().numpy()[:, fix] - wv).max() <= TOL
    others = np.setdiff1d(np.arange(T), fix)
    assert np.array_equal(got_k[:, others], ctx_k[:, others])


@pytest.mark.parametrize("D", [8, 32, 64, 128, 256])
def test_attention_entry_points_agree(D):
    """tdkv_attention (one context, one CTA per row) and tdkv_attention_many
    (per-row CTAs, the 8-row two-pass tiles, the 16-row online-softmax tiles,
    the 64-row register-blocked tiles and the 128-row tensor-core tiles)
    compute the same attention over ragged members with mixed fresh / cached
    rows (a 300-token member with 150 fixed rows spans two 128-row query
    tiles and five 64-key tiles)."""
    from paper_2604_03143_b200 import _lib
    from paper_2604_03143_b200._device import ptr, stream_handle
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(D)
    H, L, layer = 2, 2, 1
    hid = H * D
    Ts, fixes = [37, 90, 5, 300], []
    for T in Ts:
        n = T // 2 if T >= 300 else max(1, T // 3)
        fixes.append(np.sort(rng.choice(T, n, replace=False)).astype(np.int64))
    F = [f.size for f in fixes]
    R = sum(F)
    row0 = np.concatenate([[0], np.cumsum(F)[:-1]])
    q = torch.randn(R, hid, device=dev)
    kf = torch.randn(R, hid, device=dev)
    vf = torch.randn(R, hid, device=dev)
    ctx = [(torch.randn(L, T, hid, device=dev), torch.randn(L, T, hid, device=dev)) for T in Ts]
    fresh_of = []
    for T, f in zip(Ts, fixes):
        fo = np.full(T, -1, np.int32)
        fo[f] = np.arange(f.size, dtype=np.int32)
        fresh_of.append(torch.from_numpy(fo).to(dev))
    d_fix = [torch.from_numpy(f).to(dev) for f in fixes]
    scale = float(np.float32(1.0 / np.sqrt(D)))
    stream = stream_handle(dev)
    want = torch.empty(R, hid, device=dev)
    for i in range(len(Ts)):
        sl = slice(int(row0[i]), int(row0[i]) + F[i])
        _lib.call("tdkv_attention", ptr(q[sl]), ptr(kf[sl]), ptr(vf[sl]), ptr(ctx[i][0][layer]),
                  ptr(ctx[i][1][layer]), ptr(fresh_of[i]), ptr(d_fix[i]), F[i], Ts[i], H, D,
                  scale, ptr(want[sl]), stream)
    forms = [(0, 8)] + ([(8, 8), (16, 16)] if D <= 128 else [])   # (tile rows, rows arg)
    forms += [(64, 64)] if D in (8, 16, 32, 64, 128) else []
    forms += [(128, 128)] if D in (32, 64) else []
    for tile, rows_arg in forms:
        members = np.zeros(len(Ts), _lib.ATTN_MEMBER)
        tiles = -(-np.asarray(F) // max(tile, 1)) if tile else np.zeros(len(Ts), np.int64)
        tile0 = np.concatenate([[0], np.cumsum(tiles)[:-1]])
        for i in range(len(Ts)):
            members[i] = (ptr(ctx[i][0]), ptr(ctx[i][1]), ptr(fresh_of[i]), ptr(d_fix[i]),
                          Ts[i] * hid, int(row0[i]), F[i], Ts[i], int(tile0[i]))
        d_members = torch.from_numpy(members.view(np.uint8)).to(dev)
        got = torch.full((R, hid), float("nan"), device=dev)
        _lib.call("tdkv_attention_many", ptr(q), ptr(kf), ptr(vf), ptr(d_members), len(Ts), layer,
                  R, int(tiles.sum()), rows_arg, max(Ts), H, D, scale, ptr(got), stream)
        torch.cuda.synchronize()
        assert torch.isfinite(got).all()
        # the online softmax rescales per tile: equal up to float rounding;
        # the tensor-core tiles multiply in 3xTF32 (~22 mantissa bits)
        tol = {16: 2e-6, 64: 2e-6, 128: 5e-6}.get(tile, 1e-6)
        assert (got - want).abs().max().item() <= tol, tile

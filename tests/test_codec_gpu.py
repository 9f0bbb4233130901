"""GPU parity of the single-shard codec kernels (K1 diff, K4 apply, reslice,
copy_overlap, extract, generator) against the oracle, through the C-ABI.

Bar: bit-exact indices, values and patched weights.  The checkers are the
C restatement (oracle/wsync_oracle.c) and, for F32/I32, the compiled
reference itself (oracle/_ref)."""
import numpy as np
import pytest
import torch

from oracle.oracle import BF16, F32, I32

pytestmark = pytest.mark.gpu

NP = {BF16: np.uint16, I32: np.int32, F32: np.float32}
TD = {BF16: torch.bfloat16, I32: torch.int32, F32: torch.float32}


def to_dev(a, dt):
    t = torch.from_numpy(np.ascontiguousarray(a).view({BF16: np.int16, I32: np.int32,
                                                       F32: np.float32}[dt]).copy())
    if dt == BF16:
        t = t.view(torch.bfloat16)
    return t.cuda()


def to_np(t, dt):
    t = t.detach().cpu()
    if dt == BF16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def rand_pair(rng, dt, n, density):
    if dt == F32:
        prev = rng.uniform(-1, 1, n).astype(np.float32)
        nxt = prev.copy()
        m = rng.random(n) < density
        nxt[m] += (0.5 + rng.random(m.sum())).astype(np.float32)
        # +0/-0 corner case (value compare, codec.cpp:46); NaN has its own test
        if n > 4:
            prev[0], nxt[0] = 0.0, -0.0
    elif dt == I32:
        prev = rng.integers(-2**31, 2**31 - 1, n, dtype=np.int64).astype(np.int32)
        nxt = prev.copy()
        m = rng.random(n) < density
        nxt[m] = (nxt[m].astype(np.int64) + rng.integers(1, 2**31, m.sum())).astype(np.int32)
    else:
        prev = rng.integers(0, 1 << 16, n).astype(np.uint16)
        nxt = prev.copy()
        m = rng.random(n) < density
        nxt[m] += rng.integers(1, 1 << 16, m.sum()).astype(np.uint16)
    return prev, nxt


SIZES = [0, 1, 7, 8, 9, 4095, 4096, 4097, 8191, 8192, 8193, 65536 + 3, 1_000_003]


@pytest.mark.parametrize("dt", [BF16, I32, F32])
@pytest.mark.parametrize("n", SIZES)
def test_diff_matches_oracle(restatement, dt, n):
    import paper_2605_06534_b200 as ws
    rng = np.random.default_rng(n * 7 + dt)
    for density in (0.0, 0.01, 0.3, 1.0):
        prev, nxt = rand_pair(rng, dt, n, density)
        want_i, want_v = restatement.diff_shards(dt, prev, nxt)
        d = ws.diff_shards(to_dev(prev, dt), to_dev(nxt, dt))
        got_i = to_np(d.indices, I32).view(np.uint32)
        assert got_i.tolist() == want_i.tolist(), (n, density)
        assert to_np(d.values, dt).tobytes() == want_v.tobytes()


def test_diff_nan_and_signed_zero_follow_reference(reference):
    """F32 compares by value: +0 -> -0 is not a change, NaN -> NaN is (codec.cpp:46)."""
    import paper_2605_06534_b200 as ws
    prev = np.array([0.0, np.nan, 1.0, 2.0], np.float32)
    nxt = np.array([-0.0, np.nan, 1.0, 3.0], np.float32)
    ri, rv = reference.diff_shards(F32, [4], prev, nxt)
    d = ws.diff_shards(to_dev(prev, F32), to_dev(nxt, F32))
    assert to_np(d.indices, I32).tolist() == ri.tolist() == [1, 3]
    # NaN payloads differ between x86 and the GPU; only the non-NaN value is compared bitwise
    assert to_np(d.values, F32)[1] == rv[1] == 1.0


@pytest.mark.parametrize("dt", [BF16, I32, F32])
def test_diff_cap_counts_all_writes_prefix(restatement, dt):
    """Records past `cap` are counted but not written (the density fallback)."""
    import paper_2605_06534_b200 as ws
    rng = np.random.default_rng(3)
    prev, nxt = rand_pair(rng, dt, 100_000, 0.5)
    want_i, _ = restatement.diff_shards(dt, prev, nxt)
    cap = 1000
    d = ws.diff_shards(to_dev(prev, dt), to_dev(nxt, dt), cap=cap)
    assert d.nnz() == cap
    assert to_np(d.indices, I32).tolist() == want_i[:cap].tolist()


@pytest.mark.parametrize("dt", [BF16, I32, F32])
def test_apply_matches_oracle(restatement, dt):
    import paper_2605_06534_b200 as ws
    rng = np.random.default_rng(11)
    prev, nxt = rand_pair(rng, dt, 32 * 16 * 37, 0.1)
    idx, val = restatement.diff_shards(dt, prev, nxt)
    want, rc = restatement.apply_delta(dt, prev, idx, val)
    assert rc == 0
    tgt = to_dev(prev, dt)
    delta = ws.SparseDelta(dt, (prev.size,), torch.from_numpy(idx.astype(np.int32)).cuda(),
                           to_dev(val, dt).view({BF16: torch.int16, I32: torch.int32,
                                                 F32: torch.float32}[dt]))
    ws.apply_delta(tgt, delta)
    assert to_np(tgt, dt).tobytes() == want.tobytes()
    if dt != F32:
        assert to_np(tgt, dt).tobytes() == nxt.tobytes()


def test_apply_out_of_shard_leaves_target_untouched():
    """Deliberate tightening of codec.cpp:73-79: validate before any write."""
    import paper_2605_06534_b200 as ws
    tgt = torch.arange(16, dtype=torch.int32, device="cuda")
    delta = ws.SparseDelta(I32, (16,), torch.tensor([1, 4, 99, 5], dtype=torch.int32,
                                                    device="cuda"),
                           torch.ones(4, dtype=torch.int32, device="cuda"))
    with pytest.raises(ws.IndexOutOfShard):
        ws.apply_delta(tgt, delta)
    assert tgt.cpu().tolist() == list(range(16))
    with pytest.raises(ws.ShapeMismatch):
        ws.apply_delta(torch.zeros(8, dtype=torch.int32, device="cuda"), delta)


def test_reslice_kats():
    """transfer_test.cpp:297-354 through the GPU kernel."""
    import paper_2605_06534_b200 as ws
    vals = torch.tensor([10, 20, 30], dtype=torch.int32, device="cuda")
    full = (6, 4)
    cases = [((0, 2, 4), (0, 3, 6), (2, 4), [1, 5, 7], [1, 3], [20, 30]),
             ((1, 0, 4), (1, 2, 4), (6, 4), [0, 3, 23], [1, 11], [20, 30]),
             ((-1, 0, 0), (0, 3, 6), (6, 4), [0, 3, 23], [11], [30]),
             ((0, 2, 4), (-1, 0, 0), (2, 4), [1, 5, 7], [9, 13, 15], [10, 20, 30])]
    for src, dst, dshape, idx, wi, wv in cases:
        d = ws.SparseDelta(I32, dshape, torch.tensor(idx, dtype=torch.int32, device="cuda"), vals)
        out = ws.reslice_delta(d, src, dst, full, allow_cross_dim=False)
        assert out.indices.cpu().tolist() == wi
        assert out.values.cpu().tolist() == wv
        assert out.shape == ws.shard_shape(full, dst)
    bad = ws.SparseDelta(I32, (2, 4), torch.tensor([1, 5, 100], dtype=torch.int32,
                                                   device="cuda"), vals)
    with pytest.raises(ws.IndexOutOfShard):
        ws.reslice_delta(bad, (0, 2, 4), (0, 3, 6), full)
    with pytest.raises(ws.ShapeMismatch):
        ws.reslice_delta(ws.SparseDelta(I32, (3, 4), bad.indices, vals), (0, 2, 4), (0, 3, 6), full)
    with pytest.raises(ws.ShapeMismatch):
        ws.reslice_delta(ws.SparseDelta(I32, (2, 4), bad.indices[:1], vals[:1]), (0, 2, 4),
                         (1, 0, 2), full, allow_cross_dim=False)


@pytest.mark.parametrize("seed", range(8))
def test_reslice_matches_reference_and_restatement(reference, restatement, seed):
    import paper_2605_06534_b200 as ws
    from oracle.oracle import shard_shape
    rng = np.random.default_rng(500 + seed)
    nd = int(rng.integers(1, 4))
    full = [int(rng.integers(1, 6)) * 4 for _ in range(nd)]

    def desc(dim):
        if rng.random() < 0.2:
            return (-1, 0, 0)
        parts = int(rng.choice([1, 2, 4]))
        r = int(rng.integers(0, parts))
        per = full[dim] // parts
        return (dim, per * r, per * (r + 1))

    sd = int(rng.integers(0, nd))
    same = rng.random() < 0.5 or nd == 1
    dd = sd if same else int((sd + 1) % nd)
    src, dst = desc(sd), desc(dd)
    sshape = shard_shape(full, src)
    n = int(np.prod(sshape))
    idx = np.flatnonzero(rng.random(n) < rng.uniform(0, 1)).astype(np.uint64)
    val = rng.integers(-1000, 1000, idx.size).astype(np.int32)
    wi, wv = restatement.reslice_delta(I32, full, src, dst, idx, val, allow_cross_dim=True)
    cross = src[0] >= 0 and dst[0] >= 0 and src[0] != dst[0]
    if not cross:
        ri, rv, _ = reference.reslice_delta(I32, full, src, dst, sshape, idx, val)
        assert ri.tolist() == wi.tolist()
    d = ws.SparseDelta(I32, tuple(sshape), torch.from_numpy(idx.astype(np.int32)).cuda(),
                       torch.from_numpy(val).cuda())
    out = ws.reslice_delta(d, src, dst, full)
    assert out.indices.cpu().numpy().astype(np.uint64).tolist() == wi.tolist()
    assert out.values.cpu().numpy().tobytes() == wv.tobytes()


@pytest.mark.parametrize("dt", [BF16, I32])
def test_extract_and_copy_overlap_match_oracle(restatement, dt):
    import paper_2605_06534_b200 as ws
    rng = np.random.default_rng(21)
    full = [12, 16, 8]
    n = int(np.prod(full))
    full_np = rand_pair(rng, dt, n, 0.0)[0]
    full_t = to_dev(full_np, dt).view(*full)
    descs = [(-1, 0, 0), (0, 4, 8), (1, 0, 8), (1, 8, 16), (2, 2, 6), (0, 0, 12)]
    for d in descs:
        got = ws.extract_shard(full_t, d)
        assert to_np(got, dt).ravel().tobytes() == \
            restatement.extract_shard(dt, full_np, full, d).tobytes()
    for sd in descs:
        for dd in descs:
            src = restatement.extract_shard(dt, full_np, full, sd)
            dst0 = np.zeros(int(np.prod(ws.shard_shape(full, dd))), NP[dt])
            want, wn = restatement.copy_overlap_box(dt, full, dd, dst0, sd, src)
            dst_t = to_dev(dst0, dt).view(*ws.shard_shape(full, dd))
            got_n = ws.copy_overlap(dst_t, dd, to_dev(src, dt).view(*ws.shard_shape(full, sd)),
                                    sd, full)
            assert got_n == wn
            assert to_np(dst_t, dt).ravel().tobytes() == want.tobytes(), (sd, dd)


def test_copy_overlap_same_dim_matches_reference(reference):
    """shard.cpp:136-170 (transfer_test.cpp:118-145)."""
    import paper_2605_06534_b200 as ws
    full = np.arange(24, dtype=np.int32)
    src = full.reshape(6, 4)[3:6].ravel().copy()
    rd, rn = reference.copy_overlap(I32, [2, 4], np.zeros(8, np.int32), 2, [3, 4], src, 3, 0)
    dst_t = torch.zeros(2, 4, dtype=torch.int32, device="cuda")
    n = ws.copy_overlap(dst_t, (0, 2, 4), torch.from_numpy(src).cuda().view(3, 4), (0, 3, 6),
                        (6, 4))
    assert n == rn == 4
    assert dst_t.cpu().numpy().ravel().tolist() == rd.tolist()


@pytest.mark.parametrize("desc", [(-1, 0, 0), (0, 8, 24), (1, 32, 64)])
def test_generator_matches_oracle(restatement, desc):
    import paper_2605_06534_b200 as ws
    full = (48, 64)
    p, n = ws.gen_pair_bf16(3, "layers.0.w", full, desc, 0.05)
    wp, wn = restatement.gen_pair_bf16(3, "layers.0.w", full, desc, 0.05)
    assert to_np(p, BF16).ravel().tobytes() == wp.tobytes()
    assert to_np(n, BF16).ravel().tobytes() == wn.tobytes()


@pytest.mark.parametrize("desc", [(-1, 0, 0), (0, 4, 12), (2, 32, 64)])
def test_skewed_generator_matches_oracle(restatement, desc):
    """Config 4: per-expert change thresholds along dim 0 of a stacked expert tensor."""
    import paper_2605_06534_b200 as ws
    full = (16, 8, 64)
    thr = ws.expert_thresholds(16, 0.05, 1.1, 5)
    p, n = ws.gen_pair_bf16(3, "layers.0.mlp.experts.up_proj", full, desc, 0.0, thr_dim0=thr)
    wp, wn = restatement.gen_pair_bf16(3, "layers.0.mlp.experts.up_proj", full, desc, 0.0,
                                       thr_dim0=thr)
    assert to_np(p, BF16).ravel().tobytes() == wp.tobytes()
    assert to_np(n, BF16).ravel().tobytes() == wn.tobytes()
    assert (wp != wn).any()

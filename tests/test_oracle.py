"""Pins the C restatement (oracle/wsync_oracle.c) to the compiled reference.

CPU only.  Every check here compares the restatement with the unmodified
reference (oracle/_ref/libref_capi.so, built from
/root/reference/proj/src/transfer) or with the known-answer vectors of the
reference's own tests (proj/tests/transfer_test.cpp, cited per test).
BF16 has no reference counterpart; it is pinned by running the reference's
I32 path on zero-extended 16-bit words (the low 16 bits of a u32 wrap-around
difference/sum are the u16 wrap-around difference/sum).
"""
import numpy as np
import pytest

from oracle.oracle import BF16, F32, I32, OracleError, shard_shape


def _rand_pair(rng, dtype, n, density):
    if dtype == F32:
        prev = rng.uniform(-1, 1, n).astype(np.float32)
        nxt = prev.copy()
        m = rng.random(n) < density
        nxt[m] += (0.5 + rng.random(m.sum())).astype(np.float32)
    elif dtype == I32:
        prev = rng.integers(-1000, 1001, n).astype(np.int32)
        nxt = prev.copy()
        m = rng.random(n) < density
        nxt[m] += rng.integers(1, 101, m.sum()).astype(np.int32)
    else:
        prev = rng.integers(0, 1 << 16, n).astype(np.uint16)
        nxt = prev.copy()
        m = rng.random(n) < density
        nxt[m] += rng.integers(1, 1 << 16, m.sum()).astype(np.uint16)
    return prev, nxt


# --- known-answer vectors of the reference's own tests -----------------------

def test_kat_diff(restatement, reference):
    # transfer_test.cpp:207-224: I32 iota 4x4, +7 at 3, -2 at 9
    prev = np.arange(16, dtype=np.int32)
    nxt = prev.copy()
    nxt[3] += 7
    nxt[9] -= 2
    for idx, val in (restatement.diff_shards(I32, prev, nxt),
                     reference.diff_shards(I32, [4, 4], prev, nxt)):
        assert idx.tolist() == [3, 9]
        assert val.tolist() == [7, -2]
    assert restatement.diff_shards(I32, prev, prev)[0].size == 0


def test_kat_reslice(restatement, reference):
    # transfer_test.cpp:297-354
    full = [6, 4]
    vals = np.array([10, 20, 30], np.int32)
    cases = [
        ((0, 2, 4), (0, 3, 6), [2, 4], [1, 5, 7], [1, 3], [20, 30]),
        ((1, 0, 4), (1, 2, 4), [6, 4], [0, 3, 23], [1, 11], [20, 30]),
        ((-1, 0, 0), (0, 3, 6), [6, 4], [0, 3, 23], [11], [30]),
        ((0, 2, 4), (-1, 0, 0), [2, 4], [1, 5, 7], [9, 13, 15], [10, 20, 30]),
    ]
    for src, dst, dshape, idx, want_idx, want_val in cases:
        oi, ov = restatement.reslice_delta(I32, full, src, dst, np.array(idx, np.uint64),
                                           vals, allow_cross_dim=False)
        ri, rv, rshape = reference.reslice_delta(I32, full, src, dst, dshape,
                                                 np.array(idx, np.uint64), vals)
        assert oi.tolist() == want_idx == ri.tolist()
        assert ov.tolist() == want_val == rv.tolist()
        assert rshape == shard_shape(full, dst)
    # out-of-shard index -> IndexOutOfShard in both (transfer_test.cpp:349-350)
    with pytest.raises(OracleError) as e:
        restatement.reslice_delta(I32, full, (0, 2, 4), (0, 3, 6),
                                  np.array([1, 5, 100], np.uint64), vals)
    assert e.value.kind == "IndexOutOfShard"
    with pytest.raises(OracleError) as e:
        reference.reslice_delta(I32, full, (0, 2, 4), (0, 3, 6), [2, 4],
                                np.array([1, 5, 100], np.uint64), vals)
    assert e.value.kind == "IndexOutOfShard"
    # cross-dim slices are rejected by the reference (codec.cpp:101-102)
    with pytest.raises(OracleError) as e:
        reference.reslice_delta(I32, full, (0, 2, 4), (1, 0, 2), [2, 4],
                                np.array([1], np.uint64), vals[:1])
    assert e.value.kind == "ShapeMismatch"
    with pytest.raises(OracleError) as e:
        restatement.reslice_delta(I32, full, (0, 2, 4), (1, 0, 2),
                                  np.array([1], np.uint64), vals[:1], allow_cross_dim=False)
    assert e.value.kind == "ShapeMismatch"


def test_kat_extract_and_overlap(restatement, reference):
    # transfer_test.cpp:90-145
    t = np.arange(24, dtype=np.int32)
    r = restatement.extract_shard(I32, t, [4, 6], (0, 1, 3))
    assert r[0] == 6 and r[11] == 17
    c = restatement.extract_shard(I32, t, [4, 6], (1, 2, 5))
    assert c[0] == 2 and c[3] == 8 and c[11] == 22
    for desc in ((0, 1, 3), (1, 2, 5), (-1, 0, 0), (1, 0, 6)):
        assert (restatement.extract_shard(I32, t, [4, 6], desc)
                == reference.extract_shard(I32, t, [4, 6], desc)).all()
    with pytest.raises(OracleError):
        restatement.extract_shard(I32, t, [4, 6], (0, 1, 9))
    with pytest.raises(OracleError):
        reference.extract_shard(I32, t, [4, 6], (0, 1, 9))
    # partial overlap: dst rows [2,4) of a [6,4] tensor, src rows [3,6)
    full = np.arange(24, dtype=np.int32)
    src = restatement.extract_shard(I32, full, [6, 4], (0, 3, 6))
    dst, n = restatement.copy_overlap_box(I32, [6, 4], (0, 2, 4),
                                          np.zeros(8, np.int32), (0, 3, 6), src)
    assert n == 4 and dst[4] == 12 and dst[0] == 0
    rdst, rn = reference.copy_overlap(I32, [2, 4], np.zeros(8, np.int32), 2, [3, 4], src, 3, 0)
    assert rn == n and (rdst == dst).all()


# --- randomized restatement-vs-reference parity ------------------------------

@pytest.mark.parametrize("dtype", [F32, I32])
@pytest.mark.parametrize("seed", range(4))
def test_diff_apply_match_reference(restatement, reference, dtype, seed):
    rng = np.random.default_rng(seed)
    shape = [int(rng.integers(1, 40)), int(rng.integers(1, 40))]
    n = shape[0] * shape[1]
    prev, nxt = _rand_pair(rng, dtype, n, float(rng.uniform(0, 0.6)))
    oi, ov = restatement.diff_shards(dtype, prev, nxt)
    ri, rv = reference.diff_shards(dtype, shape, prev, nxt)
    assert (oi == ri).all() and oi.tobytes() == ri.tobytes()
    assert ov.tobytes() == rv.tobytes()
    a, rc = restatement.apply_delta(dtype, prev, oi, ov)
    b, rc2 = reference.apply_delta(dtype, shape, prev, shape, ri, rv)
    assert rc == rc2 == 0 and a.tobytes() == b.tobytes()
    if dtype == I32:
        assert a.tobytes() == nxt.tobytes()  # exact dtype reconstructs next


def test_apply_out_of_shard_matches_reference(restatement, reference):
    # transfer_test.cpp:240-243: both stop with IndexOutOfShard, partially applied
    prev = np.arange(16, dtype=np.int32)
    idx = np.array([1, 4, 99, 5], np.uint64)
    val = np.array([1, 1, 1, 1], np.int32)
    a, rc = restatement.apply_delta(I32, prev, idx, val)
    b, rc2 = reference.apply_delta(I32, [4, 4], prev, [4, 4], idx, val)
    assert rc == rc2 == 3
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("seed", range(12))
def test_reslice_same_dim_matches_reference(restatement, reference, seed):
    rng = np.random.default_rng(100 + seed)
    nd = int(rng.integers(1, 4))
    full = [int(rng.integers(1, 5)) * 4 for _ in range(nd)]
    dim = int(rng.integers(0, nd))

    def desc():
        if rng.random() < 0.25:
            return (-1, 0, 0)
        parts = int(rng.choice([1, 2, 4]))
        r = int(rng.integers(0, parts))
        per = full[dim] // parts
        return (dim, per * r, per * (r + 1))

    src, dst = desc(), desc()
    sshape = shard_shape(full, src)
    n = int(np.prod(sshape))
    dens = float(rng.uniform(0.0, 1.0))
    idx = np.flatnonzero(rng.random(n) < dens).astype(np.uint64)
    val = rng.integers(-1000, 1000, idx.size).astype(np.int32)
    oi, ov = restatement.reslice_delta(I32, full, src, dst, idx, val, allow_cross_dim=False)
    ri, rv, _ = reference.reslice_delta(I32, full, src, dst, sshape, idx, val)
    assert oi.tolist() == ri.tolist()
    assert ov.tobytes() == rv.tobytes()


@pytest.mark.parametrize("seed", range(6))
def test_cross_dim_reslice_matches_dense_reconstruction(restatement, seed):
    """the cross-dim oracle is dense arithmetic on the full tensor."""
    rng = np.random.default_rng(200 + seed)
    full = [8, 12, 3][: int(rng.integers(2, 4))]
    a, b = 0, 1
    src = (a, 2, 6)
    dst = (b, 4, 12)
    sshape = shard_shape(full, src)
    prev_full = rng.integers(-5, 5, int(np.prod(full))).astype(np.int32)
    nxt_full = prev_full.copy()
    m = rng.random(prev_full.size) < 0.3
    nxt_full[m] += 1
    ps = restatement.extract_shard(I32, prev_full, full, src)
    ns = restatement.extract_shard(I32, nxt_full, full, src)
    idx, val = restatement.diff_shards(I32, ps, ns)
    assert int(np.prod(sshape)) == ps.size
    oi, ov = restatement.reslice_delta(I32, full, src, dst, idx, val)
    assert (np.diff(oi.astype(np.int64)) > 0).all()  # stays ascending
    tgt = restatement.extract_shard(I32, prev_full, full, dst)
    got, rc = restatement.apply_delta(I32, tgt, oi, ov)
    assert rc == 0
    # dense reconstruction: take next inside the src box, prev elsewhere
    want_full = prev_full.reshape(full).copy()
    sl = [slice(None)] * len(full)
    sl[a] = slice(src[1], src[2])
    want_full[tuple(sl)] = nxt_full.reshape(full)[tuple(sl)]
    want = restatement.extract_shard(I32, want_full.ravel(), full, dst)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("seed", range(4))
def test_bf16_is_the_reference_i32_rule_on_u16_words(restatement, reference, seed):
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(1, 3000))
    prev, nxt = _rand_pair(rng, BF16, n, float(rng.uniform(0, 0.5)))
    oi, ov = restatement.diff_shards(BF16, prev, nxt)
    ri, rv = reference.diff_shards(I32, [n], prev.astype(np.int32), nxt.astype(np.int32))
    assert oi.tolist() == ri.tolist()
    assert ov.tolist() == (rv.view(np.uint32) & 0xFFFF).astype(np.uint16).tolist()
    got, rc = restatement.apply_delta(BF16, prev, oi, ov)
    rgot, rc2 = reference.apply_delta(I32, [n], prev.astype(np.int32), [n], ri,
                                      ov.astype(np.int32))
    assert rc == rc2 == 0
    assert got.tolist() == (rgot.view(np.uint32) & 0xFFFF).astype(np.uint16).tolist()
    assert got.tobytes() == nxt.tobytes()


def test_density_rule(restatement):
    # engine.cpp:121: inclusive threshold
    assert restatement.is_sparse(20, 100, 0.20)
    assert not restatement.is_sparse(21, 100, 0.20)
    assert restatement.is_sparse(0, 0, 0.20)


def test_sparse_payload_matches_reference(restatement, reference):
    # codec.cpp:164-183 / transfer_test.cpp:248-270: the I32/F32 wire bytes
    rng = np.random.default_rng(9)
    prev, nxt = _rand_pair(rng, I32, 24, 0.3)
    idx, val = restatement.diff_shards(I32, prev, nxt)
    for iw in (4, 8):
        assert restatement.encode_sparse(I32, [8, 3], idx, val, iw) == \
            reference.encode_sparse(I32, [8, 3], idx, val, iw)


def test_generator_is_layout_independent(restatement):
    full = [16, 24]
    p_full, n_full = restatement.gen_pair_bf16(5, "w", full, (-1, 0, 0), 0.1)
    for desc in ((0, 4, 12), (1, 6, 18)):
        p, n = restatement.gen_pair_bf16(5, "w", full, desc, 0.1)
        assert p.tobytes() == restatement.extract_shard(BF16, p_full, full, desc).tobytes()
        assert n.tobytes() == restatement.extract_shard(BF16, n_full, full, desc).tobytes()
    frac = (p_full != n_full).mean()
    assert 0.03 < frac < 0.2

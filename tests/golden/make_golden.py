#!/usr/bin/env python
"""Generates tests/golden/reference_vectors.npz from the COMPILED, unmodified
reference (oracle/_ref/libref_capi.so, built by oracle/Makefile from
/root/reference/proj/src/transfer) -- run here, where /root/reference
exists; the fixture is committed so parity stays pinned on hosts without it
(the GPU boxes).

    python tests/golden/make_golden.py      # rewrites reference_vectors.npz

Contents (every array produced by the reference's own functions):
  diff/<dtype>/<k>     codec.cpp:34-63 diff_shards + codec.cpp:65-92 apply_delta
  bf16/<k>             the same on 16-bit words (the reference's I32 path on
                       zero-extended words, low 16 bits)
  reslice/<k>          codec.cpp:94-138 reslice_delta (same-dim, randomized)
  wire/<dtype>/<iw>    codec.cpp:145-183 encode_sparse / encode_dense payloads
  key/<k>, frame/<k>   key.cpp:47-69 BucketKey::encode, wire.cpp:35-47 frames
  sync/<layout>        engine.cpp:66-254 TransferEngine::sync_step on a toy
                       model (I32): both snapshots, every serving rank's
                       weights afterwards, the report's shard counts/bytes
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import F32, I32, Reference, shard_shape  # noqa: E402

OUT = os.path.join(HERE, "reference_vectors.npz")

# toy layouts for the sync vectors: (train tp, pp, dp) -> (serve tp, pp)
SYNC_LAYOUTS = {"tp2-tp2": ((2, 1, 1), (2, 1)), "tp2pp2-tp1pp2": ((2, 2, 1), (1, 2)),
                "tp1dp2-tp1": ((1, 1, 2), (1, 1)), "tp4-tp2": ((4, 1, 1), (2, 1))}


def rand_pair(rng, dtype, n, density):
    if dtype == F32:
        prev = rng.uniform(-1, 1, n).astype(np.float32)
        nxt = prev.copy()
        m = rng.random(n) < density
        nxt[m] += (0.5 + rng.random(m.sum())).astype(np.float32)
    else:
        prev = rng.integers(-1000, 1001, n).astype(np.int32)
        nxt = prev.copy()
        m = rng.random(n) < density
        nxt[m] += rng.integers(1, 101, m.sum()).astype(np.int32)
    return prev, nxt


def generate(ref):
    g = {}
    rng = np.random.default_rng(2605)
    for dtype in (F32, I32):
        for k, (shape, dens) in enumerate((([7, 9], 0.3), ([64, 48], 0.01), ([3, 5, 40], 0.15),
                                           ([1, 1], 1.0), ([500], 0.0))):
            n = int(np.prod(shape))
            prev, nxt = rand_pair(rng, dtype, n, dens)
            idx, val = ref.diff_shards(dtype, shape, prev, nxt)
            tgt = (prev + (1 if dtype == I32 else np.float32(0.25))).astype(prev.dtype)
            applied, rc = ref.apply_delta(dtype, shape, tgt, shape, idx, val)
            assert rc == 0
            p = f"diff/{dtype}/{k}/"
            g.update({p + "shape": np.array(shape, np.int64), p + "prev": prev, p + "next": nxt,
                      p + "idx": idx.astype(np.uint64), p + "val": val, p + "target": tgt,
                      p + "applied": applied})
    # bf16 has no reference code: the reference's I32 path on zero-extended
    # 16-bit words (the low 16 bits of its u32 wrap-around delta / sum are the
    # u16 wrap-around delta / sum)
    for k, (n, dens) in enumerate(((4099, 0.01), (777, 0.3), (64, 1.0))):
        prev = rng.integers(0, 1 << 16, n).astype(np.uint16)
        nxt = prev.copy()
        m = rng.random(n) < dens
        nxt[m] += rng.integers(1, 1 << 16, m.sum()).astype(np.uint16)
        prev[:4] = [0x7FC1, 0x0000, 0x8000, 0xFF80]  # NaN payload, +0, -0, -inf by bits
        nxt[:4] = [0x7FC2, 0x8000, 0x8000, 0x7F80]
        idx, val = ref.diff_shards(I32, [n], prev.astype(np.int32), nxt.astype(np.int32))
        tgt = rng.integers(0, 1 << 16, n).astype(np.uint16)
        applied, rc = ref.apply_delta(I32, [n], tgt.astype(np.int32), [n], idx, val)
        assert rc == 0
        p = f"bf16/{k}/"
        g.update({p + "prev": prev, p + "next": nxt, p + "idx": idx.astype(np.uint64),
                  p + "val": (val.astype(np.int64) & 0xFFFF).astype(np.uint16),
                  p + "target": tgt, p + "applied": (applied.astype(np.int64) & 0xFFFF).astype(
                      np.uint16)})
    for k in range(10):
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
        idx = np.flatnonzero(rng.random(n) < rng.uniform(0, 1)).astype(np.uint64)
        val = rng.integers(-1000, 1000, idx.size).astype(np.int32)
        oi, ov, oshape = ref.reslice_delta(I32, full, src, dst, sshape, idx, val)
        p = f"reslice/{k}/"
        g.update({p + "full": np.array(full, np.int64), p + "src": np.array(src, np.int64),
                  p + "dst": np.array(dst, np.int64), p + "idx": idx, p + "val": val,
                  p + "out_idx": np.asarray(oi, np.uint64), p + "out_val": np.asarray(ov, np.int32),
                  p + "out_shape": np.array(oshape, np.int64)})
    for dtype in (F32, I32):
        shape = [48, 64]
        prev, nxt = rand_pair(rng, dtype, 48 * 64, 0.05)
        idx, val = ref.diff_shards(dtype, shape, prev, nxt)
        p = f"wire/{dtype}/"
        g[p + "shape"] = np.array(shape, np.int64)
        g[p + "idx"] = idx.astype(np.uint64)
        g[p + "val"] = val
        g[p + "next"] = nxt
        for iw in (4, 8):
            g[p + f"sparse{iw}"] = np.frombuffer(ref.encode_sparse(dtype, shape, idx, val, iw),
                                                 np.uint8)
        g[p + "dense"] = np.frombuffer(ref.encode_dense(dtype, shape, nxt), np.uint8)
    keys = [(7, "model.layers.0.self_attn.q_proj.weight", 1, 2, 0, (0, 64, 128), "S", 4, 0),
            (123456789, "lm_head.weight", 0, 1, 1, (-1, 0, 0), "D", 0, 3),
            (1, "a/b c%dé", 3, 4, 1, (1, 8, 16), "S", 8, 12)]
    for k, args in enumerate(keys):
        key = ref.bucket_key(*args)
        payload = rng.integers(0, 256, int(rng.integers(0, 3000)), dtype=np.uint8).tobytes()
        frame = ref.encode_bucket_frame(key, payload)
        p = f"key/{k}/"
        g.update({p + "step": np.array([args[0]], np.uint64),
                  p + "param": np.frombuffer(args[1].encode("utf-8"), np.uint8),
                  p + "ints": np.array([args[2], args[3], args[4], *args[5], args[7], args[8]],
                                       np.int64),
                  p + "codec": np.frombuffer(args[6].encode(), np.uint8),
                  p + "key": np.frombuffer(key, np.uint8),
                  p + "payload": np.frombuffer(payload, np.uint8),
                  p + "frame": np.frombuffer(frame, np.uint8),
                  p + "crc": np.array([ref.frame_crc32(payload)], np.uint64)})
    for name, (train, serve) in SYNC_LAYOUTS.items():
        st = ref.toy_state(2, 32, 64, I32, train, serve, 0.05, 11)
        p = f"sync/{name}/"
        g[p + "train"] = np.array(train, np.int64)
        g[p + "serve"] = np.array(serve, np.int64)
        g[p + "params"] = np.array([f"{n}|{k}|{'x'.join(map(str, s))}|{l}"
                                    for (n, k, s, l) in st.params])
        for i in range(len(st.params)):
            g[p + f"prev/{i}"] = st.weights(i, 0, I32)
            g[p + f"next/{i}"] = st.weights(i, 1, I32)
        rep = st.run(mode_async=True, shard_aware=True, sparse=True, threshold=0.20,
                     bucket_bytes=8192)
        g[p + "report"] = np.array([rep["dense_shards"], rep["sparse_shards"],
                                    rep["pushed_bytes"]], np.int64)
        coords = serve[0] * serve[1]
        for c in range(coords):
            for i in range(len(st.params)):
                w = st.serve(c, i, I32)
                if w is not None:
                    g[p + f"serve/{c}/{i}"] = w
    return g


def main():
    g = generate(Reference())
    np.savez_compressed(OUT, **g)
    print(f"{OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()

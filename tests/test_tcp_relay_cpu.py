"""The framed client of the test harness against the reference's own
TcpRelayServer (tcp_relay.hpp:10-17), on the CPU: a frame built by the
reference's encode_bucket_frame (wire.cpp:35-47) is stored after PUT, comes
back from GET_ANY byte for byte, and a flipped bit in transit is rejected by
the server's CRC check (status 3).  The GPU tests (test_relay.py) then send
GPU-built frames through the same path."""
import ctypes as C

import numpy as np


def _put(tcp, frame: bytes):
    fn = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64)(tcp.callbacks[3])
    buf = np.frombuffer(frame, np.uint8).copy()
    return fn(tcp.ctx, buf.ctypes.data, len(frame))


def _get_any(tcp, keys, cap=1 << 20):
    fn = C.CFUNCTYPE(C.c_int64, C.c_void_p, C.POINTER(C.c_char_p), C.POINTER(C.c_uint64), C.c_int,
                     C.c_int, C.POINTER(C.c_int), C.c_void_p, C.c_uint64)(tcp.callbacks[4])
    kb = [k.encode() for k in keys]
    ka = (C.c_char_p * len(kb))(*kb)
    la = (C.c_uint64 * len(kb))(*[len(k) for k in kb])
    hit = C.c_int(-1)
    out = np.empty(cap, np.uint8)
    n = fn(tcp.ctx, ka, la, len(kb), 500, C.byref(hit), out.ctypes.data, cap)
    return n, hit.value, out[:max(n, 0)].tobytes()


def test_framed_put_and_get_any_through_reference_server(reference):
    tcp = reference.tcp_relay()
    payload = bytes(range(256)) * 40
    frame = reference.encode_bucket_frame(b"w|s1|pa|q0", payload)
    assert _put(tcp, frame) == 0
    assert tcp.buckets() == 1 and tcp.get("w|s1|pa|q0") == payload
    n, hit, got = _get_any(tcp, ["w|s1|pb|q0", "w|s1|pa|q0"])
    assert hit == 1 and got == frame
    n, hit, got = _get_any(tcp, ["w|s1|missing"])
    assert n == -1  # timeout
    tcp.close()


def test_flipped_bit_is_rejected_by_the_server_crc(reference):
    tcp = reference.tcp_relay(flip_put=1)
    frame = reference.encode_bucket_frame(b"w|s1|px|q0", b"\x07" * 1000)
    assert _put(tcp, frame) == 3  # tcp_relay.hpp: status 3, integrity failure
    assert tcp.buckets() == 0
    tcp.close()

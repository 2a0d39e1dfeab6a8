"""CPU: the host half of the wire layer (paper_2003_05328_b200/wire.py) against the
compiled reference (oracle/_ref): config digest, Hello/Done/Error frames and REF's
decode_frame checks, FNV transcript hashing, in-process and TCP transports."""
import struct
import threading

import numpy as np
import pytest
import torch

import oracle as O
from conftest import fnv
from paper_2003_05328_b200 import protocol as GP
from paper_2003_05328_b200 import wire as W

Q = 576460803525083137
P = 638977
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _sched(desc):
    return [GP.Conv(d[1], d[2], bool(d[3]), d[4], d[5]) if d[0] == 0 else GP.Act(d[6]) for d in desc]


def test_fnv1a_matches_reference_definition():
    rng = np.random.default_rng(1)
    for n in (0, 1, 7, 4096):
        b = rng.integers(0, 256, size=n, dtype=np.uint8).tobytes()
        h = 1469598103934665603
        for x in b:
            h = ((h ^ x) * 1099511628211) & ((1 << 64) - 1)
        assert W.fnv1a(b) == h
    # chained over u64 LE words == the fixtures' digest helper
    x = rng.integers(0, 2**63, size=64, dtype=np.uint64)
    assert "%016x" % W.fnv1a(x.astype("<u8").tobytes()) == fnv(x)


@needs_ref
def test_config_digest_vs_reference(golden):
    cases = [(c["seed"], c["H"], c["W"], c["n"], c["mode"], c["desc"]) for c in golden["proto"]]
    cases += [(5, 16, 8, 4096, 0, [[0, 3, 1, 0, 2, 4, 0], [1, 0, 0, 0, 0, 0, 1], [0, 1, 1, 1, 4, 4, 0]])]
    for seed, H, Wd, n, mode, desc in cases:
        ref = O.ref().ref_config_digest(P, Q, n, 4.0, mode, seed, H, Wd, len(desc),
                                        np.array(desc, np.int32).reshape(-1))
        assert W.config_digest(n, Q, P, seed, H, Wd, _sched(desc), freq_direct=bool(mode)) == ref


def _ref_share_frame(layer, v):
    out = np.zeros(W.FRAME_HEADER_BYTES + 16 + 8 * v.size + 8, np.uint8)
    ln = O.C.c_size_t()
    ch, r, c = v.shape
    assert O.ref().ref_wire_share_frame(W.ACTIVATION_SHARE_UP, layer, ch, r, c,
                                        np.ascontiguousarray(v.reshape(-1), np.uint64), out.ctypes.data,
                                        out.size, O.C.byref(ln)) == 0
    return out[:ln.value].tobytes()


def _ref_decode_kind(frame: bytes, expect=W.ACTIVATION_SHARE_UP, shape=(1, 2, 2)):
    buf = np.frombuffer(frame, np.uint8).copy() if frame else np.zeros(1, np.uint8)
    layer = O.C.c_uint32()
    v = np.zeros(max(1, int(np.prod(shape))), np.uint64)
    rc = O.ref().ref_wire_share_decode(buf.ctypes.data, len(frame), expect, *shape, P, O.C.byref(layer), v)
    return {0: None, 14: "MalformedPayload", 12: "ProtocolOrderViolation"}[rc], O.ref().ref_last_error().decode()


@needs_ref
def test_host_frame_checks_match_reference():
    """check_frame / expect_host raise what REF decode_frame + recv_expect raise."""
    good = _ref_share_frame(3, np.arange(4, dtype=np.uint64).reshape(1, 2, 2))
    assert W.check_frame(good) == W.ACTIVATION_SHARE_UP
    bad = {
        "short": good[:10],
        "magic": b"X" + good[1:],
        "version": good[:4] + b"\x02" + good[5:],
        "type0": good[:5] + b"\x00" + good[6:],
        "type8": good[:5] + b"\x08" + good[6:],
        "cap": good[:6] + struct.pack("<Q", (1 << 30) + 1) + good[14:],
        "length": good[:-1],
        "error": W.error_frame("boom"),
        "unexpected": W.done_frame(),
    }
    for name, f in bad.items():
        kind, msg = _ref_decode_kind(f)
        with pytest.raises(W.EnseiError) as e:
            W.expect_host(f, W.ACTIVATION_SHARE_UP)
        assert e.value.kind == kind, name
        assert msg in str(e.value), (name, msg, str(e.value))


def test_hello_done_frames_layout():
    h = W.hello_frame(0x0123456789ABCDEF)
    assert h[:6] == b"ENSE\x01\x01" and struct.unpack("<Q", h[6:14])[0] == 8
    assert struct.unpack("<Q", W.expect_host(h, W.HELLO))[0] == 0x0123456789ABCDEF
    d = W.done_frame()
    assert len(d) == W.FRAME_HEADER_BYTES and W.expect_host(d, W.DONE) == b""


def test_recording_inproc_transcript():
    a, b = W.make_inproc_pair()
    ra, rb = W.RecordingTransport(a), W.RecordingTransport(b)
    frames = [W.hello_frame(7), W.encode_frame(W.ACTIVATION_SHARE_UP, bytes(range(40))), W.done_frame()]
    for f in frames:
        ra.send_frame(f)
    got = [rb.recv_frame() for _ in frames]
    assert got == frames
    h = W.FNV_OFFSET
    for f in frames:
        h = W.fnv1a(f, h)
    assert ra.transcript.content_hash_sent == h == rb.transcript.content_hash_recv
    assert ra.transcript.total_bytes("sent") == sum(len(f) for f in frames)
    assert rb.transcript.total_bytes("recv", W.HELLO) == 22
    a.close()
    with pytest.raises(W.TransportError):
        b.recv_frame()


def test_tcp_transport_roundtrip_and_header_validation():
    port = 46000 + (np.random.default_rng().integers(0, 2000))
    ready = threading.Event()
    box = {}

    def server():
        try:
            t = W.TcpTransport.listen_and_accept(int(port), ready=ready)
            box["frames"] = [t.recv_frame()]
            buf = torch.zeros(200, dtype=torch.uint8)
            box["into"] = bytes(t.recv_frame_into(buf).numpy())
            try:
                t.recv_frame()
            except W.EnseiError as e:
                box["err"] = e.kind
            t.close()
        except Exception as e:  # noqa: BLE001
            box["fail"] = e
            ready.set()

    th = threading.Thread(target=server)
    th.start()
    ready.wait(10)
    c = W.TcpTransport.connect("127.0.0.1", int(port))
    f1 = W.hello_frame(42)
    f2 = W.encode_frame(W.ACTIVATION_SHARE_DOWN, bytes(range(100)))
    c.send_frame(f1)
    c.send_frame(torch.frombuffer(bytearray(f2), dtype=torch.uint8))
    c.send_frame(b"XNSE\x01\x01" + bytes(8))
    th.join(10)
    c.close()
    assert "fail" not in box, box.get("fail")
    assert box["frames"] == [f1] and box["into"] == f2 and box["err"] == "MalformedPayload"

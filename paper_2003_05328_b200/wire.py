"""Wire framing and transports: the reference's message layer over the device path.

REF: wire.hpp:17-80 / wire.cpp (frames, ciphertext records, transports, transcript
hashing) and protocol.cpp:55-150 (recv_expect, encode/decode_ct_blocks,
encode/decode_shares, config_digest).

Ciphertext-block and share frames -- the bulk of every transcript -- are built and
parsed by kernels (ensei_gpu_wire_*) straight from / into the device layouts,
reading and writing page-locked host buffers in place, so a frame never takes a
host serialisation pass.  The tiny Hello / Done / Error frames are built here.
Transports carry encoded frames (bytes-like); a RecordingTransport chains REF's
FNV-1a over every frame exactly as REF's RecordingTransport does (wire.cpp:336-352),
so transcript hashes are comparable with the reference's.
"""
from __future__ import annotations

import ctypes as C
import queue
import socket
import struct
import threading
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from ._lib import EnseiError, check, lib

# REF MsgType (wire.hpp:17-25)
HELLO, CIPHERTEXT_BLOCKS, ALICE_SHARE_CIPHERTEXTS = 0x01, 0x02, 0x03
ACTIVATION_SHARE_UP, ACTIVATION_SHARE_DOWN, DONE, ERROR = 0x04, 0x05, 0x06, 0x07
MSG_NAMES = {1: "Hello", 2: "CiphertextBlocks", 3: "AliceShareCiphertexts", 4: "ActivationShareUp",
             5: "ActivationShareDown", 6: "Done", 7: "Error"}
COEFFICIENT, EVALUATION = 0, 1  # REF RingDomain (ringbfv.hpp:10)

MAGIC = b"ENSE"
VERSION = 0x01
FRAME_HEADER_BYTES = 14          # REF kFrameHeaderBytes (wire.hpp:40)
MAX_PAYLOAD_BYTES = 1 << 30      # REF kMaxPayloadBytes (wire.hpp:41)
FNV_OFFSET = 1469598103934665603


class MalformedPayload(EnseiError):
    def __init__(self, msg):
        super().__init__(14, msg)


class ProtocolOrderViolation(EnseiError):
    def __init__(self, msg):
        super().__init__(12, msg)


class TransportError(EnseiError):
    def __init__(self, msg):
        super().__init__(15, msg)


def _bytes_ptr(buf) -> C.c_void_p:
    if isinstance(buf, torch.Tensor):
        return C.c_void_p(buf.data_ptr())
    a = np.frombuffer(buf, dtype=np.uint8)
    return C.c_void_p(a.ctypes.data)


def fnv1a(buf, seed: int = FNV_OFFSET) -> int:
    """REF fnv1a (wire.cpp:409-416) over a host buffer (runs in libensei_gpu.so)."""
    n = buf.numel() if isinstance(buf, torch.Tensor) else len(buf)
    return int(lib().ensei_gpu_fnv1a(_bytes_ptr(buf), n, seed))


# ----------------------------------------------------------- host frames

def encode_frame(msg_type: int, payload: bytes = b"") -> bytes:
    """REF encode_frame (wire.cpp:44-55)."""
    if len(payload) > MAX_PAYLOAD_BYTES:
        raise MalformedPayload("payload exceeds 1 GiB cap")
    return MAGIC + bytes([VERSION, msg_type]) + struct.pack("<Q", len(payload)) + bytes(payload)


def check_frame(frame) -> int:
    """REF decode_frame's checks (wire.cpp:57-79) on an encoded frame; returns its type."""
    n = frame.numel() if isinstance(frame, torch.Tensor) else len(frame)
    if n < FRAME_HEADER_BYTES:
        raise MalformedPayload("frame shorter than header")
    hdr = bytes(frame[:FRAME_HEADER_BYTES].numpy()) if isinstance(frame, torch.Tensor) else bytes(
        frame[:FRAME_HEADER_BYTES])
    if hdr[:4] != MAGIC:
        raise MalformedPayload("bad magic")
    if hdr[4] != VERSION:
        raise MalformedPayload("unsupported version")
    if not 1 <= hdr[5] <= 7:
        raise MalformedPayload("unknown message type")
    (ln,) = struct.unpack("<Q", hdr[6:14])
    if ln > MAX_PAYLOAD_BYTES:
        raise MalformedPayload("payload length exceeds cap")
    if n != FRAME_HEADER_BYTES + ln:
        raise MalformedPayload("payload length mismatch")
    return hdr[5]


def frame_payload(frame) -> bytes:
    return bytes(frame[FRAME_HEADER_BYTES:])


def expect_host(frame, expect: int) -> bytes:
    """recv_expect (REF protocol.cpp:55-65) for a host-built frame; returns the payload."""
    t = check_frame(frame)
    if t == ERROR:
        raise ProtocolOrderViolation("peer aborted: " + frame_payload(frame).decode(errors="replace"))
    if t != expect:
        raise ProtocolOrderViolation(f"expected {MSG_NAMES[expect]}, got {MSG_NAMES[t]}")
    return frame_payload(frame)


def hello_frame(digest: int) -> bytes:
    return encode_frame(HELLO, struct.pack("<Q", digest))


def done_frame() -> bytes:
    return encode_frame(DONE)


def error_frame(msg: str) -> bytes:
    return encode_frame(ERROR, msg.encode())


# ------------------------------------------------------------ config digest

def _hash_u64(h: int, v: int) -> int:
    M = (1 << 64) - 1
    for i in range(8):
        h ^= (v >> (8 * i)) & 0xFF
        h = (h * 1099511628211) & M
    return h


def config_digest(n: int, q: int, p: int, seed: int, H: int, W: int, schedule, freq_direct: bool = True,
                  sigma: float = 4.0, p_e: Optional[int] = None, p_n: Optional[int] = None,
                  p_a: Optional[int] = None) -> int:
    """REF config_digest (protocol.cpp:211-235); schedule entries are protocol.Conv / Act."""
    h = FNV_OFFSET
    for v in (n, q, p_e or p, p_n or p, p_a or p, int(sigma * 16), 1 if freq_direct else 0, seed, H, W):
        h = _hash_u64(h, v)
    for s in schedule:
        if hasattr(s, "cin"):
            for v in (1, s.fh, s.fw, 1 if s.same else 2, s.cin, s.cout):
                h = _hash_u64(h, v)
        else:
            h = _hash_u64(_hash_u64(h, 2), s.fn)
    return h


# ---------------------------------------------------------- device frames

def ct_frame_bytes(n: int, channels: int, blocks: int) -> int:
    return int(lib().ensei_gpu_wire_ct_frame_bytes(n, channels, blocks))


def share_frame_bytes(channels: int, rows: int, cols: int) -> int:
    return int(lib().ensei_gpu_wire_share_frame_bytes(channels, rows, cols))


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def pinned_frames(num: int, nbytes: int) -> torch.Tensor:
    return torch.empty((num, nbytes), dtype=torch.uint8, pin_memory=True)


def encode_ct_blocks(ctx, msg_type: int, layer: int, ct: torch.Tensor, domain: int = EVALUATION,
                     out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """encode_frame(encode_ct_blocks(...)) (REF protocol.cpp:83-97) for every image of
    ct[img][ch][B][2][1][n] (device layout; natural coefficients when domain = Coefficient).
    Returns uint8 frames [img][frame_bytes] (page-locked host memory unless `out` given);
    asynchronous on `stream`."""
    imgs, ch, B = ct.shape[0], ct.shape[1], ct.shape[2]
    fb = ct_frame_bytes(ctx.n, ch, B)
    out = pinned_frames(imgs, fb) if out is None else out
    assert ct.dtype == torch.uint64 and ct.is_cuda and ct.is_contiguous()
    check(lib().ensei_gpu_wire_encode_ct_blocks(ctx.h, msg_type, layer, ch, B, domain, C.c_void_p(ct.data_ptr()),
                                                imgs, C.c_void_p(out.data_ptr()), out.stride(0), _stream(stream)))
    return out


def decode_ct_blocks(ctx, frames: torch.Tensor, expect_type: int, channels: int, blocks: int,
                     out: Optional[torch.Tensor] = None, stream=None):
    """recv_expect + decode_ct_blocks (REF protocol.cpp:55-65, 99-117) of frames[img][len]
    (page-locked host or device) -> (ct[img][ch][B][2][1][n] device layout, layers,
    number of Coefficient-domain records converted).  Raises the REF error."""
    imgs, ln = frames.shape
    out = torch.empty((imgs, channels, blocks, 2, 1, ctx.n), dtype=torch.uint64,
                      device=ctx.device) if out is None else out
    layers = (C.c_uint32 * max(imgs, 1))()
    ncoef = C.c_uint32(0)
    check(lib().ensei_gpu_wire_decode_ct_blocks(ctx.h, C.c_void_p(frames.data_ptr()), ln, frames.stride(0), imgs,
                                                expect_type, channels, blocks, layers, C.c_void_p(out.data_ptr()),
                                                C.byref(ncoef), _stream(stream)))
    return out, list(layers)[:imgs], ncoef.value


def encode_shares(ctx, msg_type: int, layer: int, shares: torch.Tensor, out: Optional[torch.Tensor] = None,
                  stream=None) -> torch.Tensor:
    """encode_frame(encode_shares(...)) (REF protocol.cpp:119-132) of shares[img][ch][rows][cols]
    (int32/uint32 residues, device) -> uint8 frames [img][frame_bytes]."""
    imgs, ch, rows, cols = shares.shape
    fb = share_frame_bytes(ch, rows, cols)
    out = pinned_frames(imgs, fb) if out is None else out
    assert shares.is_cuda and shares.is_contiguous() and shares.element_size() == 4
    check(lib().ensei_gpu_wire_encode_shares(ctx.h, msg_type, layer, ch, rows, cols, C.c_void_p(shares.data_ptr()),
                                             imgs, C.c_void_p(out.data_ptr()), out.stride(0), _stream(stream)))
    return out


def decode_shares(ctx, frames: torch.Tensor, expect_type: int, channels: int, rows: int, cols: int,
                  max_value: int, out: Optional[torch.Tensor] = None, stream=None):
    """recv_expect + decode_shares (REF protocol.cpp:134-150) -> (int32 shares
    [img][ch][rows][cols] on the device, layers)."""
    imgs, ln = frames.shape
    out = torch.empty((imgs, channels, rows, cols), dtype=torch.int32, device=ctx.device) if out is None else out
    layers = (C.c_uint32 * max(imgs, 1))()
    check(lib().ensei_gpu_wire_decode_shares(ctx.h, C.c_void_p(frames.data_ptr()), ln, frames.stride(0), imgs,
                                             expect_type, channels, rows, cols, max_value, layers,
                                             C.c_void_p(out.data_ptr()), _stream(stream)))
    return out, list(layers)[:imgs]


# ---------------------------------------------------------------- transports

class Transport:
    """REF Transport (wire.hpp): frames are encoded bytes-like objects."""

    def send_frame(self, frame) -> None:
        raise NotImplementedError

    def recv_frame(self):
        raise NotImplementedError


class _Queue:
    def __init__(self):
        self.q: "queue.Queue" = queue.Queue()
        self.closed = False


class InprocTransport(Transport):
    """One end of REF make_inproc_pair (wire.cpp:168-230): frames are validated on receipt."""

    def __init__(self, tx: _Queue, rx: _Queue):
        self.tx, self.rx = tx, rx

    def send_frame(self, frame) -> None:
        self.tx.q.put(frame)

    def recv_frame(self):
        while True:
            try:
                f = self.rx.q.get(timeout=0.1)
                break
            except queue.Empty:
                if self.rx.closed:
                    raise TransportError("peer closed")
        check_frame(f)
        return f

    def close(self) -> None:
        self.tx.closed = True


def make_inproc_pair():
    ab, ba = _Queue(), _Queue()
    return InprocTransport(ab, ba), InprocTransport(ba, ab)


class TcpTransport(Transport):
    """REF TcpTransport (wire.cpp:232-321): one frame = header + payload on a stream
    socket; the header is validated before the length is trusted.  recv_frame can land
    the frame straight in a caller's page-locked buffer (recv_frame_into)."""

    def __init__(self, sock: socket.socket):
        self.sock = sock
        self.sock.setsockopt(socket.IPPROTO_TCP, socket.TCP_NODELAY, 1)

    @classmethod
    def listen_and_accept(cls, port: int, host: str = "127.0.0.1", ready: Optional[threading.Event] = None):
        srv = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
        srv.setsockopt(socket.SOL_SOCKET, socket.SO_REUSEADDR, 1)
        try:
            srv.bind((host, port))
            srv.listen(1)
            if ready is not None:
                ready.set()
            fd, _ = srv.accept()
        except OSError as e:
            raise TransportError(f"listen/accept failed: {e}")
        finally:
            srv.close()
        return cls(fd)

    @classmethod
    def connect(cls, host: str, port: int, retries: int = 50):
        for attempt in range(retries + 1):
            s = socket.socket(socket.AF_INET, socket.SOCK_STREAM)
            try:
                s.connect((host, port))
                return cls(s)
            except OSError:
                s.close()
                if attempt >= retries:
                    raise TransportError("connect() failed")
                time.sleep(0.1)

    def close(self) -> None:
        self.sock.close()

    def send_frame(self, frame) -> None:
        mv = memoryview(frame.numpy() if isinstance(frame, torch.Tensor) else frame).cast("B")
        try:
            self.sock.sendall(mv)
        except OSError:
            raise TransportError("send() failed")

    def _recv_exact(self, mv: memoryview) -> None:
        got = 0
        while got < len(mv):
            k = self.sock.recv_into(mv[got:])
            if k <= 0:
                raise TransportError("recv() failed or peer closed")
            got += k

    def _header(self) -> int:
        hdr = bytearray(FRAME_HEADER_BYTES)
        self._recv_exact(memoryview(hdr))
        if bytes(hdr[:4]) != MAGIC:
            raise MalformedPayload("bad magic")
        if hdr[4] != VERSION:
            raise MalformedPayload("unsupported version")
        if not 1 <= hdr[5] <= 7:
            raise MalformedPayload("unknown message type")
        (ln,) = struct.unpack("<Q", bytes(hdr[6:14]))
        if ln > MAX_PAYLOAD_BYTES:
            raise MalformedPayload("payload length exceeds cap")
        return hdr, ln

    def recv_frame(self):
        hdr, ln = self._header()
        buf = bytearray(FRAME_HEADER_BYTES + ln)
        buf[:FRAME_HEADER_BYTES] = hdr
        self._recv_exact(memoryview(buf)[FRAME_HEADER_BYTES:])
        return bytes(buf)

    def recv_frame_into(self, out: torch.Tensor) -> torch.Tensor:
        """Receive one frame into the uint8 host tensor `out` (e.g. a row of a pinned
        batch buffer); returns the filled prefix."""
        hdr, ln = self._header()
        total = FRAME_HEADER_BYTES + ln
        if total > out.numel():
            raise MalformedPayload("payload length mismatch")
        mv = memoryview(out.numpy()).cast("B")
        mv[:FRAME_HEADER_BYTES] = hdr
        self._recv_exact(mv[FRAME_HEADER_BYTES:total])
        return out[:total]


@dataclass
class Transcript:
    """REF Transcript (wire.hpp): FNV-1a chains and byte counts per direction."""
    content_hash_sent: int = FNV_OFFSET
    content_hash_recv: int = FNV_OFFSET
    entries: List[tuple] = field(default_factory=list)  # (direction 'sent'/'recv', type, bytes)

    def total_bytes(self, direction: str, msg_type: Optional[int] = None) -> int:
        return sum(b for d, t, b in self.entries if d == direction and (msg_type is None or t == msg_type))


def _frame_type(frame) -> int:
    return int(frame[5])


class RecordingTransport(Transport):
    """REF RecordingTransport (wire.cpp:336-352)."""

    def __init__(self, inner: Transport):
        self.inner = inner
        self.transcript = Transcript()

    def send_frame(self, frame) -> None:
        self.inner.send_frame(frame)
        t = self.transcript
        t.content_hash_sent = fnv1a(frame, t.content_hash_sent)
        t.entries.append(("sent", _frame_type(frame), len(frame)))

    def recv_frame(self):
        f = self.inner.recv_frame()
        t = self.transcript
        t.content_hash_recv = fnv1a(f, t.content_hash_recv)
        t.entries.append(("recv", _frame_type(f), len(f)))
        return f


def gather_frames(frames: Sequence, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Stack received frames (equal length) into one page-locked [num][len] batch for the
    device decoder (one host copy; TcpTransport.recv_frame_into lands there directly)."""
    lens = {len(f) for f in frames}
    if len(lens) != 1:
        # different lengths: each frame is decoded against its own length by the caller
        raise MalformedPayload("payload length mismatch")
    ln = lens.pop()
    out = pinned_frames(len(frames), ln) if out is None else out
    dst = out.numpy()
    for i, f in enumerate(frames):
        src = f.numpy() if isinstance(f, torch.Tensor) else np.frombuffer(f, dtype=np.uint8)
        dst[i, :ln] = src
    return out

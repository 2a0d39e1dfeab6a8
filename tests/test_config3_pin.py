"""CPU: config 3's plaintext ground truth (oracle/protocol.py plain_protocol, the
checker the GPU stack tests use) equals the compiled reference's own
reference_pipeline (REF protocol.cpp:694-750) on each of the three
reference-expressible segments of the seven-layer stack, at the
real channel counts.  The 2x2 max-pool between segments is the builder's extension
and is applied outside REF, on the centered lift, exactly as plain_protocol does."""
import numpy as np
import pytest

import oracle as O
from oracle import protocol as OP
from paper_2003_05328_b200 import configs as CF

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _oracle_sched(sched):
    return [OP.Conv(s.fh, s.fw, s.same, s.cin, s.cout) if hasattr(s, "cin") else OP.Act(s.fn, s.pool2) for s in sched]


def _ref_pipeline(sched, img, ws):
    rows = np.array(OP.desc_rows(sched), np.int32).reshape(-1)
    cout = [s for s in sched if isinstance(s, OP.Conv)][-1].cout
    H = img.shape[1]
    out = np.zeros(cout * H * H, np.uint64)
    O.ref_check(O.ref().ref_reference_pipeline(CF.P, CF.Q, 2048, H, H, len(sched), rows,
                                               np.ascontiguousarray(img, np.int64).reshape(-1),
                                               np.concatenate([w.reshape(-1) for w in ws]).astype(np.int64), out))
    return out.reshape(cout, H, H)


@pytest.mark.parametrize("seg", [0, 1, 2])
def test_config3_segment_vs_reference_pipeline(seg):
    lo, hi, side, cin = CF.CONFIG3_SEGMENTS[seg]
    sched = _oracle_sched(CF.CONFIG3_SCHEDULE[lo:hi])
    rng = np.random.default_rng(300 + seg)
    # segment inputs: pixels for the first, pooled residues mod p (full range) after that
    img = rng.integers(0, 256 if seg == 0 else CF.P, size=(cin, side, side)).astype(np.int64)
    convs = [i for i, s in enumerate(CF.CONFIG3_SCHEDULE) if hasattr(s, "cin")]
    ws = [rng.integers(-128, 128, size=CF.CONFIG3_WEIGHTS[convs.index(i)]).astype(np.int64)
          for i in range(lo, hi) if i in convs]
    want = _ref_pipeline(sched, img, ws)
    got = OP.plain_protocol(sched, img, ws, CF.Q, CF.P, 2048, OP.default_workers())
    assert (got == want).all()


def test_config3_pool_is_max_of_centered_lifts():
    p = CF.P
    x = np.array([[[1, p - 1], [5, p - 7]]], np.uint64)  # lifts 1, -1, 5, -7 -> max 5
    got = OP.plain_protocol([OP.Act(2, True)], x.astype(np.int64), [], CF.Q, p, 2048)
    assert got.reshape(-1).tolist() == [5]
    y = np.array([[[p - 3, p - 1], [p - 9, p - 2]]], np.uint64)  # all negative -> -1
    got = OP.plain_protocol([OP.Act(2, True)], y.astype(np.int64), [], CF.Q, p, 2048)
    assert got.reshape(-1).tolist() == [p - 1]

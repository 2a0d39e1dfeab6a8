"""GPU: a two-PROCESS session over TCP -- Bob in a child process (tests/tcp_party.py),
Alice here, each with its own CUDA context, frames built / parsed by the wire kernels
straight from / into page-locked buffers and sent over a localhost socket.  Parity
mode with REF's randomness (product RefRng): both transcripts equal the reference's
golden transcript hashes (tests/golden/golden.json)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import fnv
from gpu_util import dev, to_np

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("idx", [0, 2])
def test_two_process_tcp_session_matches_reference(golden, tmp_path, idx):
    from paper_2003_05328_b200 import ops, protocol, refrand, schedule, wire
    case = golden["proto"][idx]
    layers = [{"kind": "conv", "filter_h": d[1], "filter_w": d[2], "conv_type": "same" if d[3] else "valid",
               "channels_in": d[4], "channels_out": d[5]} if d[0] == 0 else
              {"kind": "activation", "fn": schedule.FN_NAME[d[6]]} for d in case["desc"]]
    (tmp_path / "schedule.json").write_text(json.dumps({"layers": layers}))
    sf = schedule.load_schedule_file(str(tmp_path / "schedule.json"))
    H, W, n, seed = case["H"], case["W"], case["n"], case["seed"]
    g = refrand.RefRng(seed, 0xDA7A)  # REF's fixture draws (tests/golden/make_golden.py)
    cin = sf.schedule[0].cin
    img = g.uniform_below(256, cin * H * W).astype(np.int64).reshape(cin, H, W)
    convs = [s for s in sf.schedule if isinstance(s, protocol.Conv)]
    ws = [(g.uniform_below(256, s.cout * s.cin * s.fh * s.fw).astype(np.int64) - 128).reshape(s.cout, s.cin, s.fh, s.fw)
          for s in convs]
    for i, w in enumerate(ws):
        np.save(tmp_path / f"w{i}.npy", w)
    (tmp_path / "session.json").write_text(json.dumps({"n": n, "H": H, "W": W, "seed": seed, "convs": len(ws),
                                                       "freq_direct": case["mode"]}))
    port = _free_port()
    bob = subprocess.Popen([sys.executable, os.path.join(HERE, "tcp_party.py"), "bob", str(port), str(tmp_path)],
                           stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
    try:
        ctx = ops.Context(n=n)
        sess = protocol.Session(ctx, sf.schedule, H, W, [torch.from_numpy(w.astype(np.int32)) for w in ws])
        sr = refrand.SessionRandomness(ctx, [seed])
        key = sr.keys()[0]
        rnd = sr.for_session(sess)
        rands = [rnd(li) for li in range(len(sf.schedule))]
        digest = wire.config_digest(n, ctx.q[0], ctx.p, seed, H, W, sf.schedule, bool(case["mode"]))
        t = wire.TcpTransport.connect("127.0.0.1", port, retries=600)
        x = torch.from_numpy(img.astype(np.int32)[None]).to(dev())
        alice = protocol.run_alice(sess, key, x, rands, [t], digest, bool(case["mode"]))
        t.close()
        out, err = bob.communicate(timeout=300)
    finally:
        if bob.poll() is None:
            bob.kill()
    assert bob.returncode == 0, err[-2000:]
    b = json.loads(out.strip().splitlines()[-1])
    ta = alice.transcripts[0]
    assert "%016x" % ta.content_hash_sent == case["alice_sent"] == b["recv"]
    assert "%016x" % ta.content_hash_recv == case["alice_recv"] == b["sent"]
    assert ta.total_bytes("sent") == case["alice_bytes_sent"] and b["bytes_sent"] == case["bob_bytes_sent"]
    assert fnv(to_np(alice.output).astype(np.uint64).reshape(-1)) == case["out_fnv"]
    order = ["ct_ntt", "ring_ntt", "image_ntt", "hadamard"]
    assert [b["counters"][k] for k in order] == case["counters_bob"]

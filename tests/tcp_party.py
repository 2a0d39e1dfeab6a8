"""Helper process for tests/test_gpu_tcp.py: one party of a session over TCP, product
code only (schedule.py, refrand.py, protocol.py, wire.py).  Prints its transcript as JSON.

    python tests/tcp_party.py bob PORT WORKDIR
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2003_05328_b200 import ops, protocol, refrand, schedule, wire  # noqa: E402


def main():
    role, port, work = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    cfg = json.load(open(os.path.join(work, "session.json")))
    sf = schedule.load_schedule_file(os.path.join(work, "schedule.json"))
    ws = [np.load(os.path.join(work, f"w{i}.npy")) for i in range(cfg["convs"])]
    ctx = ops.Context(n=cfg["n"])
    sess = protocol.Session(ctx, sf.schedule, cfg["H"], cfg["W"], [torch.from_numpy(w.astype(np.int32)) for w in ws])
    sr = refrand.SessionRandomness(ctx, [cfg["seed"]])
    rnd = sr.for_session(sess)
    digest = wire.config_digest(ctx.n, ctx.q[0], ctx.p, cfg["seed"], cfg["H"], cfg["W"], sf.schedule,
                                bool(cfg["freq_direct"]))
    assert role == "bob"
    t = wire.TcpTransport.listen_and_accept(port)
    rands = [rnd(li) for li in range(len(sf.schedule))]
    res = protocol.run_bob(sess, rands, [t], digest)
    t.close()
    tr = res.transcripts[0]
    print(json.dumps({"sent": "%016x" % tr.content_hash_sent, "recv": "%016x" % tr.content_hash_recv,
                      "bytes_sent": tr.total_bytes("sent"), "counters": res.counters}), flush=True)


if __name__ == "__main__":
    main()

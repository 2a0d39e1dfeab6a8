"""Config-2 kernel driver for ncu: batched negacyclic forward + inverse (device layout)
over 65536 polynomials of degree n (default 2048).  `python tools/profile_ntt.py [n] [reps]`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2003_05328_b200 import _lib, ops  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
Q = 576460803525083137
ctx = ops.Context(n=n)
buf = torch.randint(0, 1 << 62, (65536, n), dtype=torch.int64, device="cuda")
buf = (buf % Q).view(torch.uint64)
for _ in range(reps):
    ctx.negacyclic(buf, 0, False, _lib.LAYOUT_BITREV)
    ctx.negacyclic(buf, 0, True, _lib.LAYOUT_BITREV)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    ctx.negacyclic(buf, 0, False, _lib.LAYOUT_BITREV)
b.record()
b.synchronize()
print("fwd ms", a.elapsed_time(b) / 5)

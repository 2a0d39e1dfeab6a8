import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2003_05328_b200 import ops, _lib
from paper_2003_05328_b200.configs import Q
for n, cnt in ((2048, 65536), (4096, 32768), (8192, 16384)):
    ctx = ops.Context(n=n, q=(Q,))
    buf = torch.randint(0, 2**59, (cnt, n), dtype=torch.int64, device='cuda').view(torch.uint64)
    buf = (buf.view(torch.int64) % Q).view(torch.uint64)
    for inv in (False, True):
        for _ in range(3): ctx.negacyclic(buf, 0, inv, _lib.LAYOUT_BITREV)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): ctx.negacyclic(buf, 0, inv, _lib.LAYOUT_BITREV)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(n, 'inv' if inv else 'fwd', round(cnt / ms / 1e3, 2), 'M transforms/s')

"""Helpers for the -m gpu tests (oracle on the CPU side as the checker)."""
import numpy as np
import torch

import oracle as O
from oracle import protocol as OP

Q = 576460803525083137
P = 638977
RNS = (576460803525083137, 576461033843064833, 576461054781063169)


def dev():
    return torch.device("cuda", 0)


def to_np(t):
    return t.detach().cpu().numpy()


def u64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64)).to(dev())


def bitrev_perm(n):
    bits = n.bit_length() - 1
    return np.array([int(format(i, f"0{bits}b")[::-1], 2) for i in range(n)])


def golden_inputs(case):
    g = O.MTRng(case["seed"], 0xDA7A)
    convs = [d for d in case["desc"] if d[0] == 0]
    H, W = case["H"], case["W"]
    img = np.array([g.uniform_below(256) for _ in range(convs[0][4] * H * W)], np.int64).reshape(convs[0][4], H, W)
    ws = [np.array([g.uniform_below(256) - 128 for _ in range(d[1] * d[2] * d[4] * d[5])], np.int64)
          .reshape(d[5], d[4], d[1], d[2]) for d in convs]
    sched = [OP.Conv(d[1], d[2], bool(d[3]), d[4], d[5]) if d[0] == 0 else OP.Act(d[6]) for d in case["desc"]]
    return img, ws, sched

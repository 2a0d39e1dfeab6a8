"""BASELINE.json's five workloads as data (shapes and parameters only; the inputs are
seeded synthetic draws -- no dataset).  Used by bench.py and the parity tests so both
run exactly the same schedules.

config 0: one 1 -> 1 3x3 Same conv of a 32x32 uint8 image, n = 2048, single prime.
config 1: one 16 -> 16 3x3 Same layer, 8 images of 16x32x32, n = 2048.
config 2: 65536 negacyclic transforms of degree 2048 / 4096 / 8192 (no layer).
config 3: seven conv layers 3->64, 64->64 @32; 64->128, 128->128 @16; 128->128 (3x3),
          128->128 (1x1), 128->16 (1x1) @8, plaintext ReLU between layers and the
          builder-defined 2x2 max-pool after layers 2 and 4, 64 images.
config 4: one 64 -> 128 3x3 Same layer, 1024 images of 64x32x32, n = 8192, RNS q of
          three 60-bit primes == 1 mod 16384 p.
"""
from __future__ import annotations

from .protocol import Act, Conv

P = 638977
Q = 576460803525083137
RNS = (576460803525083137, 576461033843064833, 576461054781063169)

CONFIG1 = dict(n=2048, q=(Q,), H=32, W=32, cin=16, cout=16, fh=3, images=8)
CONFIG4 = dict(n=8192, q=RNS, H=32, W=32, cin=64, cout=128, fh=3, images=1024)

# config 3: (schedule, weight shapes [cout][cin][fh][fw]); ReLU after every conv but the
# last, 2x2 max-pool folded into the activations after conv 2 (32 -> 16) and conv 4 (16 -> 8)
CONFIG3_SCHEDULE = [Conv(3, 3, True, 3, 64), Act(0), Conv(3, 3, True, 64, 64), Act(0, True),
                    Conv(3, 3, True, 64, 128), Act(0), Conv(3, 3, True, 128, 128), Act(0, True),
                    Conv(3, 3, True, 128, 128), Act(0), Conv(1, 1, True, 128, 128), Act(0),
                    Conv(1, 1, True, 128, 16)]
CONFIG3_WEIGHTS = [(64, 3, 3, 3), (64, 64, 3, 3), (128, 64, 3, 3), (128, 128, 3, 3), (128, 128, 3, 3),
                   (128, 128, 1, 1), (16, 128, 1, 1)]
CONFIG3_IMAGES = 64
# the same stack with every layer packing as many images per ciphertext block as the ring
# holds (1, 1, 2, 2, 8, 32, 32: the 32x32, 16x16 and 8x8 grids fill 1/2, 1/8, 1/32 of n = 2048)
CONFIG3_SCHEDULE_PACKED = [Conv(s.fh, s.fw, s.same, s.cin, s.cout, 0) if isinstance(s, Conv) else s
                           for s in CONFIG3_SCHEDULE]
# the same stack on the smallest grids dividing p - 1 = 2^14 39 that hold each layer's linear
# convolution (grid override): 39x39 for the 32x32 layers (one block per channel instead of
# two), 24x24 x 3 images for the 16x16 layers, 12x12 x 12 images for the 8x8 3x3 layer; the
# 1x1 layers keep REF's 8x8 grid x 32 images
CONFIG3_GRIDS = [(39, 1), (39, 1), (24, 3), (24, 3), (12, 12), (0, 0), (0, 0)]
CONFIG3_SCHEDULE_GRID = []
for _s in CONFIG3_SCHEDULE:
    if isinstance(_s, Conv):
        _g, _pk = CONFIG3_GRIDS[sum(isinstance(t, Conv) for t in CONFIG3_SCHEDULE_GRID)]
        CONFIG3_SCHEDULE_GRID.append(Conv(_s.fh, _s.fw, _s.same, _s.cin, _s.cout, _pk, _g))
    else:
        CONFIG3_SCHEDULE_GRID.append(_s)
CONFIG4_PACK = 2  # two 64x64 grids per n = 8192 block (REF's power-of-two grid)
# the headline geometry: the smallest grid side dividing p - 1 = 2^14 39 that holds the linear
# convolution (32 + 3 - 1 = 34 <= 39), five 39x39 grids per n = 8192 block
CONFIG4_GRID, CONFIG4_GRID_PACK = 39, 5
# the three reference-expressible segments (REF has no pooling layer): [L1, ReLU, L2] @32,
# [L3, ReLU, L4] @16, [L5, ReLU, L6, ReLU, L7] @8 as (first schedule index, last + 1, side, cin)
CONFIG3_SEGMENTS = [(0, 3, 32, 3), (4, 7, 16, 64), (8, 13, 8, 128)]

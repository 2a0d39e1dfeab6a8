"""GPU: a chain chosen by the parameter selector (params.build_params, RNS extension)
drives the device path -- a 128-channel accumulation the reference's single prime
cannot hold (REF build_params throws SearchExhausted), decrypting to the plaintext
convolution."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle as O
from gpu_util import P, dev, to_np

pytestmark = pytest.mark.gpu


def test_selected_rns_chain_runs_128_channel_accumulation():
    from paper_2003_05328_b200 import ops
    from paper_2003_05328_b200 import params as PP
    from paper_2003_05328_b200._lib import EnseiError
    prof = PP.Profile(8, 8, 3, 3)
    with pytest.raises(EnseiError, match="SearchExhausted"):
        PP.build_params(prof, 8192, accum_channels=128)  # REF's behaviour
    ps = PP.build_params(prof, 8192, accum_channels=128, max_primes=4, min_primes=3)
    assert ps.p == P and len(ps.q_primes) == 3
    ctx = ops.Context(n=ps.n, q=ps.q_primes, p=ps.p)
    rng = np.random.default_rng(8)
    cin, cout, H = 128, 2, 16  # 32x32 grid: the RNS Dec shapes (32x32 or 64x64)
    img = rng.integers(0, 256, size=(1, cin, H, H)).astype(np.uint8)
    w = rng.integers(-128, 128, size=(cout, cin, 3, 3)).astype(np.int32)
    L = ops.LayerOps(ctx, ops.ConvSpec(H, H, 3, 3, True, cin, cout))
    _, key = ops.secret_sample(ctx, 3)
    we = L.prepare_weights(torch.from_numpy(w).to(dev()))
    out = L.forward(key, we, torch.from_numpy(img).to(dev()), ops.Randomness(seed=3))
    Lo = O.layer(ps.q_primes[0], P, 2048, H, H, 3, 3, 1, cin, cout)
    direct = np.zeros(cout * H * H, np.uint64)
    O.lib().eo_conv_direct(C.byref(Lo), img[0].astype(np.uint64).reshape(-1), w.astype(np.int64).reshape(-1), direct)
    assert (to_np(out[0]).astype(np.uint64).reshape(-1) == direct).all()

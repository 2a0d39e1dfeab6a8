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


def test_crt_round_exact_at_the_boundaries():
    """The RNS decryption rounding (device fixed-point fast path + 192-bit fallback,
    ensei_gpu_crt_round = dec_rns_kernel's code) equals the oracle's exact multi-limb
    rounding (eo_crt_round) on random phi and on phi within a few units of every kind
    of rounding boundary (p phi / Q = m + 1/2 +- tiny), where the fast path must defer."""
    import ctypes as C
    import numpy as np
    import oracle as O
    from gpu_util import P, RNS, dev
    from paper_2003_05328_b200 import ops
    from paper_2003_05328_b200._lib import check, lib
    ctx = ops.Context(n=8192, q=RNS)
    Q = RNS[0] * RNS[1] * RNS[2]
    rng = np.random.default_rng(77)
    phis = [int(x) for x in rng.integers(0, 2**62, size=64)]
    phis += [(int(rng.integers(0, 2**62)) << 118) % Q for _ in range(64)]
    for m in [0, 1, 2, P // 2, P - 2, P - 1] + [int(x) for x in rng.integers(0, P, size=40)]:
        base = ((2 * m + 1) * Q) // (2 * P)  # p * base / Q just below m + 1/2
        for d in (-3, -2, -1, 0, 1, 2, 3, 4):
            phis.append((base + d) % Q)
    phis += [0, 1, Q - 1, Q // 2, Q // 2 + 1, Q // P, Q // P + 1]
    res = np.array([[ph % q for q in RNS] for ph in phis], dtype=np.uint64)
    d_res = torch.from_numpy(res).to(dev())
    d_out = torch.empty(len(phis), dtype=torch.int32, device=dev())
    check(lib().ensei_gpu_crt_round(ctx.h, C.c_void_p(d_res.data_ptr()), len(phis), C.c_void_p(d_out.data_ptr()),
                                    C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    got = d_out.cpu().numpy().astype(np.uint64)
    qs = np.array(RNS, dtype=np.uint64)
    for k, ph in enumerate(phis):
        want = O.lib().eo_crt_round(np.ascontiguousarray(res[k]), qs, 3, P)
        assert want == ((P * ph + Q // 2) // Q) % P  # the oracle itself, vs Python integers
        assert got[k] == want, (k, ph)


def test_rns_decrypt_exact_fallback_in_kernel():
    """dec_rns_kernel's own fallback: a crafted ciphertext (c0 = 0, c1 = NTT(phi)) whose
    phi puts 96 coefficients within a few units of a rounding boundary; the kernel's
    shares equal the oracle's exact decryption of the same ciphertext."""
    import ctypes as C
    import numpy as np
    import oracle as O
    from oracle import protocol as OP
    from gpu_util import P, RNS, dev
    from paper_2003_05328_b200 import ops
    from paper_2003_05328_b200._lib import LAYOUT_BITREV
    n = 8192
    ctx = ops.Context(n=n, q=RNS)
    L = ops.LayerOps(ctx, ops.ConvSpec(32, 32, 3, 3, True, 1, 1))
    _, key = ops.secret_sample(ctx, 3)
    Q = RNS[0] * RNS[1] * RNS[2]
    rng = np.random.default_rng(99)
    phi = [(int(rng.integers(0, 2**62)) << 118) % Q for _ in range(n)]
    for i in rng.choice(n, size=96, replace=False):
        m = int(rng.integers(0, P))
        phi[int(i)] = (((2 * m + 1) * Q) // (2 * P) + int(rng.integers(-3, 5))) % Q
    res = np.array([[ph % q for ph in phi] for q in RNS], dtype=np.uint64)  # coefficients [R][n]
    c1 = torch.from_numpy(res).to(dev())
    for r in range(3):
        row = c1[r:r + 1].contiguous()
        ctx.negacyclic(row, r, inverse=False, layout=LAYOUT_BITREV)
        c1[r] = row[0]
    ct = torch.zeros((1, 1, 1, 2, 3, n), dtype=torch.uint64, device=dev())
    ct[0, 0, 0, 1] = c1
    alice = L.alice_decrypt(key, ct)
    nat = ct.clone()
    ctx.permute(nat)
    Ls = OP.rns_layers(list(RNS), P, n, 32, 32, 3, 3, 1, 1, 1)
    al = np.zeros(32 * 32, np.uint64)
    te = np.zeros(3 * n, np.uint64)  # c0 = 0: the key does not enter
    arr = (O.Layer * 3)(*Ls)
    O.lib().eo_alice_decrypt_rns(C.cast(arr, C.c_void_p), 3, te, np.ascontiguousarray(nat.cpu().numpy()).reshape(-1),
                                 al)
    assert (alice.cpu().numpy().astype(np.uint64).reshape(-1) == al).all()

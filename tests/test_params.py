"""CPU: parameter selection (ensei_gpu_build_params / preset_params / min_pntt, the
restatement of REF params.cpp in libensei_gpu.so) against the compiled reference, and
the RNS extension where the reference's single prime runs out."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2003_05328_b200 import params as PP
from paper_2003_05328_b200._lib import EnseiError

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

KIND = {0: None, 3: "SearchExhausted", 11: "RangeViolation", 9: "ChainViolation", 1: "Error"}


def _ref_build(prof, n, mode, accum, floor=0, sigma=4.0):
    out = np.zeros(6, np.uint64)
    rc = O.ref().ref_build_params(prof.input_bits, prof.filter_bits, prof.f_h, prof.f_w, n, mode, accum, floor,
                                  sigma, out)
    return KIND[rc], out


PROFILES = [PP.Profile(8, 8, 3, 3), PP.Profile(8, 1, 3, 3), PP.Profile(12, 6, 3, 3), PP.Profile(8, 4, 5, 5),
            PP.Profile(2, 2, 2, 2), PP.Profile(16, 16, 1, 1), PP.Profile(20, 20, 7, 7)]


@pytest.mark.parametrize("prof", PROFILES)
@pytest.mark.parametrize("n", [16, 1024, 2048, 4096, 8192])
@pytest.mark.parametrize("mode", [PP.UNIFIED, PP.SPLIT_PAPER])
def test_build_params_matches_reference(prof, n, mode):
    for accum in (1, 16, 64, 128, 1000):
        kind, ref = _ref_build(prof, n, mode, accum)
        if kind is None:
            ps = PP.build_params(prof, n, mode, accum)
            assert (ps.p_n, ps.p_a, ps.p_e, ps.q_primes, ps.n, int(ps.insecure)) == (
                int(ref[0]), int(ref[1]), int(ref[2]), (int(ref[3]),), int(ref[4]), int(ref[5])), (prof, n, accum)
        else:
            with pytest.raises(EnseiError) as e:
                PP.build_params(prof, n, mode, accum)
            assert e.value.kind == kind, (prof, n, mode, accum, str(e.value), O.ref().ref_last_error())


def test_appendix_b_q_table_and_floor():
    # reference-derived q by accumulation count at p = 638977
    prof = PP.Profile(8, 8, 3, 3)
    ps = PP.build_params(prof, 2048, accum_channels=16)
    assert ps.p == 638977 and abs(math.log2(ps.q) - 59.43) < 0.01
    with pytest.raises(EnseiError, match="SearchExhausted"):
        PP.build_params(prof, 2048, accum_channels=128)
    kind, ref = _ref_build(prof, 2048, 0, 1, floor=1 << 21)
    ps = PP.build_params(prof, 2048, accum_channels=1, p_n_floor=1 << 21)
    assert kind is None and ps.p == int(ref[0]) and ps.q_primes[0] == int(ref[3])


@pytest.mark.parametrize("name", ["binary", "medium", "high", "toy", "bogus"])
@pytest.mark.parametrize("accum", [1, 4, 64])
def test_presets_match_reference(name, accum):
    out = np.zeros(6, np.uint64)
    rc = O.ref().ref_preset_params(name.encode(), accum, out)
    if rc == 0:
        ps = PP.preset_params(name, accum)
        assert (ps.p_n, ps.p_e, ps.q_primes[0], ps.n, int(ps.insecure)) == (
            int(out[0]), int(out[2]), int(out[3]), int(out[4]), int(out[5]))
    else:
        with pytest.raises(EnseiError) as e:
            PP.preset_params(name, accum)
        assert e.value.kind == KIND[rc]


def test_min_pntt_matches_reference():
    cases = [(8, 8, 3, 3), (12, 6, 3, 3), (0, 8, 3, 3), (8, -1, 3, 3), (33, 1, 1, 1), (32, 32, 1, 1),
             (30, 30, 3, 3), (1, 1, 1, 1)]
    import ctypes as C
    for c in cases:
        v = C.c_uint64()
        rc = O.ref().ref_min_pntt(*c, C.byref(v))
        if rc == 0:
            assert PP.min_pntt(PP.Profile(*c)) == v.value
        else:
            with pytest.raises(EnseiError) as e:
                PP.min_pntt(PP.Profile(*c))
            assert e.value.kind == KIND[rc], c


def test_rns_extension_where_reference_runs_out():
    prof = PP.Profile(8, 8, 3, 3)
    for n, accum in [(2048, 128), (2048, 1024), (8192, 128), (4096, 64)]:
        assert _ref_build(prof, n, 0, accum)[0] == "SearchExhausted"
        ps = PP.build_params(prof, n, accum_channels=accum, max_primes=4)
        assert len(ps.q_primes) >= 2
        assert math.log2(ps.q) >= ps.log2_q_min
        # minimal: dropping the last prime no longer covers the requirement
        assert math.log2(ps.q // ps.q_primes[-1]) < ps.log2_q_min
        step = 2 * n * ps.p_e
        for q in ps.q_primes:
            assert q % step == 1 and q < 1 << 62 and q >= 1 << 59
            assert pow(3, q - 1, q) == 1  # (primality is checked by the library; spot Fermat here)
        assert list(ps.q_primes) == sorted(set(ps.q_primes))
    # the BASELINE config-4 chain: three primes at n = 8192 == SURVEY Appendix B's
    ps = PP.build_params(prof, 8192, accum_channels=128, max_primes=4, min_primes=3)
    assert ps.q_primes == (576460803525083137, 576461033843064833, 576461054781063169)
    # below the cap the extension is REF's single prime
    kind, ref = _ref_build(prof, 2048, 0, 16)
    assert PP.build_params(prof, 2048, accum_channels=16, max_primes=4).q_primes == (int(ref[3]),)
    with pytest.raises(EnseiError, match="SearchExhausted"):
        PP.build_params(prof, 8192, accum_channels=1 << 63, max_primes=2)

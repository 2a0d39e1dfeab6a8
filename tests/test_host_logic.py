"""CPU: host-side logic of the product path that needs no GPU -- randomness key
derivation, stream ids, geometry rules -- against the reference / oracle."""
import numpy as np
import pytest

import oracle as O
from paper_2003_05328_b200 import ops


def test_fork_seed_matches_reference_rng_fork():
    for seed in (0, 1, 2003, 2**64 - 1):
        for salt in (0xA11CE, 0xB0B):
            assert ops.fork_seed(seed, salt) == O.lib().eo_fork_seed(seed, salt)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("H,f,same", [(32, 3, 1), (16, 3, 1), (8, 3, 1), (8, 1, 1), (12, 5, 0), (28, 5, 1)])
def test_geometry_rule_matches_reference(H, f, same):
    ph, pw = O.C.c_uint32(), O.C.c_uint32()
    O.ref_check(O.ref().ref_geometry(ops.P_DEFAULT, H, H, f, f, same, O.C.byref(ph), O.C.byref(pw)))
    L = O.layer(ops.Q_DEFAULT, ops.P_DEFAULT, 2048, H, H, f, f, same, 1, 1)
    assert (L.Lh, L.Lw) == (ph.value, pw.value)
    assert L.blocks == -(-ph.value * pw.value // 2048)


def test_bench_accounting_matches_survey_table():
    import bench
    # config 1 per image N_q = 1,409,024, N_mac = 2,097,152, N_p = 2,523,136 (batch-independent)
    k = bench.layer_counts(2048, 1, 64, 2, 16, 16, 32, 32, 32, 32, 1)
    assert sum(v["q"] for v in k.values()) == 1409024
    assert sum(v["mac"] for v in k.values()) == 2097152
    assert sum(v["p"] for v in k.values()) == 2523136

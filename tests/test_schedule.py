"""CPU: the schedule front end (REF schedule.cpp semantics) and the product's
reference-randomness stream (ensei_gpu_ref_rng_*) against the compiled reference."""
import json

import numpy as np
import pytest

import oracle as O
from paper_2003_05328_b200 import protocol as GP
from paper_2003_05328_b200 import refrand as RR
from paper_2003_05328_b200 import schedule as S
from paper_2003_05328_b200 import wire as W

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
Q = 576460803525083137
P = 638977


def _ref_draw(seed, salt, kind, bound, sigma, count):
    out = np.zeros(count, np.int64)
    O.ref_check(O.ref().ref_rng_draw(seed, salt or 0, int(salt is not None), kind, bound, sigma, count, out))
    return out


@needs_ref
@pytest.mark.parametrize("seed,salt", [(0, None), (7, 0xA11CE), (2**63 + 5, 0xB0B), (12345, 0xDA7A)])
def test_ref_rng_matches_reference(seed, salt):
    r = RR.RefRng(seed, salt)
    assert (r.next_u64(50).view(np.int64) == _ref_draw(seed, salt, 0, 0, 0, 50)).all()
    for bound in (1, 2, 3, 256, P, Q, (1 << 63) + 1):
        r = RR.RefRng(seed, salt)
        assert (r.uniform_below(bound, 300).view(np.int64) == _ref_draw(seed, salt, 1, bound, 0, 300)).all(), bound
    for sigma in (4.0, 3.2, 0.5):
        r = RR.RefRng(seed, salt)
        assert (r.gaussian(sigma, 2000) == _ref_draw(seed, salt, 2, 0, sigma, 2000)).all(), sigma


@needs_ref
def test_random_weights_matches_reference():
    desc = [[0, 3, 3, 1, 2, 3, 0], [1, 0, 0, 0, 0, 0, 0], [0, 1, 1, 0, 3, 4, 0]]
    sched = [GP.Conv(3, 3, True, 2, 3), GP.Act(0), GP.Conv(1, 1, False, 3, 4)]
    for mag, seed, salt in [(1, 3, None), (2, 9, 0x57), (128, 1, None)]:
        ref = np.zeros(2 * 3 * 9 + 3 * 4, np.int64)
        O.ref_check(O.ref().ref_random_weights(3, np.array(desc, np.int32).reshape(-1), mag, seed,
                                               int(salt is not None), salt or 0, ref))
        mine = RR.random_weights(sched, mag, RR.RefRng(seed, salt))
        assert (np.concatenate([w.reshape(-1) for w in mine]) == ref).all()
        assert max(abs(int(w.min())) for w in mine) <= mag


EXAMPLE = {"layers": [
    {"kind": "conv", "filter_h": 3, "filter_w": 3, "conv_type": "same", "channels_in": 1, "channels_out": 1},
    {"kind": "activation", "fn": "relu"}], "weights": "random", "weight_magnitude": 2}


def test_parse_documented_example_and_defaults():
    sf = S.parse_schedule(json.dumps(EXAMPLE))
    assert sf.schedule == [GP.Conv(3, 3, True, 1, 1), GP.Act(0)]
    assert sf.weights_source == "random" and sf.weight_magnitude == 2
    sf = S.parse_schedule('{"layers": [{"kind": "conv", "filter_h": 5, "filter_w": 1}, {"kind": "activation"}]}')
    assert sf.schedule == [GP.Conv(5, 1, True, 1, 1), GP.Act(2)]  # defaults: same, 1 -> 1, identity
    assert sf.weights_source == "random" and sf.weight_magnitude == 1
    sf = S.parse_schedule('{"layers": [{"kind": "conv", "filter_h": 1, "filter_w": 1, "conv_type": "valid",'
                          ' "channels_in": 4, "channels_out": 2}, {"kind": "activation", "fn": "square"}],'
                          ' "weights": "file"}')
    assert sf.schedule == [GP.Conv(1, 1, False, 4, 2), GP.Act(1)] and sf.weights_source == "file"
    assert [S.activation_name(f) for f in (0, 1, 2, 9)] == ["relu", "square", "identity", "?"]


@pytest.mark.parametrize("text,msg", [
    ("{", "schedule parse error"),
    ("[]", 'needs a "layers" array'),
    ('{"layers": 3}', 'needs a "layers" array'),
    ('{"layers": [{"kind": "pool"}]}', 'layer kind must be "conv" or "activation"'),
    ('{"layers": [{"filter_h": 3}]}', 'layer kind must be "conv" or "activation"'),
    ('{"layers": [{"kind": "conv", "filter_h": 3}]}', "conv layer needs filter_h/filter_w"),
    ('{"layers": [{"kind": "conv", "filter_h": 3, "filter_w": 3, "conv_type": "full"}]}', "unknown conv_type: full"),
    ('{"layers": [{"kind": "activation", "fn": "tanh"}]}', "unknown activation: tanh"),
    ('{"layers": [], "weights": "db"}', 'weights must be "random" or "file"'),
    ('{"layers": [], "weight_magnitude": 0}', "weight_magnitude must be >= 1"),
])
def test_parse_errors(text, msg):
    with pytest.raises(S.ScheduleError, match=msg) as e:
        S.parse_schedule(text)
    assert e.value.kind == "Error"


def test_files_and_weights(tmp_path):
    p = tmp_path / "s.json"
    p.write_text(json.dumps(EXAMPLE))
    assert S.load_schedule_file(str(p)).weight_magnitude == 2
    with pytest.raises(S.ScheduleError, match="cannot open schedule file"):
        S.load_schedule_file(str(tmp_path / "missing.json"))
    ints = tmp_path / "w.txt"
    ints.write_text("1 -2 3\n4\t5 -6\n")
    v = S.load_integers(str(ints))
    assert v.tolist() == [1, -2, 3, 4, 5, -6]
    (tmp_path / "bad.txt").write_text("1 2 x")
    with pytest.raises(S.ScheduleError, match="non-integer content"):
        S.load_integers(str(tmp_path / "bad.txt"))
    assert S.to_channel_images(v, 2, 1, 3).shape == (2, 1, 3)
    with pytest.raises(S.ScheduleError, match="wrong element count"):
        S.to_channel_images(v, 2, 2, 2)
    sched = [GP.Conv(1, 1, True, 2, 1), GP.Act(0), GP.Conv(1, 2, True, 1, 2)]
    ws = S.to_network_weights(v, sched)
    assert [w.shape for w in ws] == [(1, 2, 1, 1), (2, 1, 1, 2)]
    with pytest.raises(S.ScheduleError, match="too short"):
        S.to_network_weights(v[:5], sched)
    with pytest.raises(S.ScheduleError, match="trailing values"):
        S.to_network_weights(np.concatenate([v, v]), sched)


@needs_ref
def test_parsed_schedule_digest_matches_reference(golden):
    case = golden["proto"][2]
    layers = []
    for d in case["desc"]:
        if d[0] == 0:
            layers.append({"kind": "conv", "filter_h": d[1], "filter_w": d[2],
                           "conv_type": "same" if d[3] else "valid", "channels_in": d[4], "channels_out": d[5]})
        else:
            layers.append({"kind": "activation", "fn": S.FN_NAME[d[6]]})
    sf = S.parse_schedule(json.dumps({"layers": layers}))
    ref = O.ref().ref_config_digest(P, Q, case["n"], 4.0, case["mode"], case["seed"], case["H"], case["W"],
                                    len(case["desc"]), np.array(case["desc"], np.int32).reshape(-1))
    assert W.config_digest(case["n"], Q, P, case["seed"], case["H"], case["W"], sf.schedule) == ref

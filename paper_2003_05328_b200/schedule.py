"""Schedule front end: REF schedule.cpp (parse_schedule, load_schedule_file,
load_integers, to_channel_images, to_network_weights, activation_name) over Python's
json module -- REF parses with nlohmann::json, an un-vendored dependency absent from
the reference tree (proj/.gitignore:2), so this follows schedule.cpp's documented
format and error behaviour (schedule.hpp:19-27, schedule.cpp:29-64)."""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import List

import numpy as np

from ._lib import EnseiError
from .protocol import Act, Conv

RANDOM, FILE = "random", "file"  # REF WeightsSource
FN = {"relu": 0, "square": 1, "identity": 2}  # REF ActivationFn order
FN_NAME = {v: k for k, v in FN.items()}


class ScheduleError(EnseiError):
    """REF ensei::Error raised by the schedule front end."""

    def __init__(self, msg: str):
        super().__init__(1, msg)


@dataclass
class ScheduleFile:
    """REF ScheduleFile (schedule.hpp:12-17)."""
    schedule: List = field(default_factory=list)
    weights_source: str = RANDOM
    weight_magnitude: int = 1


def _int(layer: dict, key: str, default: int) -> int:
    v = layer.get(key, default)
    if isinstance(v, bool) or not isinstance(v, int):
        raise ScheduleError(f"schedule field {key!r} must be an integer")
    if v < 0:
        raise ScheduleError(f"schedule field {key!r} must be non-negative")
    return v


def _str(layer: dict, key: str, default: str) -> str:
    v = layer.get(key, default)
    if not isinstance(v, str):
        raise ScheduleError(f"schedule field {key!r} must be a string")
    return v


def parse_schedule(text: str) -> ScheduleFile:
    """REF parse_schedule (schedule.cpp:29-64)."""
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise ScheduleError(f"schedule parse error: {e}")
    if not isinstance(doc, dict) or not isinstance(doc.get("layers"), list):
        raise ScheduleError('schedule needs a "layers" array')
    out = ScheduleFile()
    for l in doc["layers"]:
        if not isinstance(l, dict):
            raise ScheduleError('layer kind must be "conv" or "activation"')
        kind = _str(l, "kind", "")
        if kind == "conv":
            fh, fw = _int(l, "filter_h", 0), _int(l, "filter_w", 0)
            ct = _str(l, "conv_type", "same")
            if ct not in ("same", "valid"):
                raise ScheduleError("unknown conv_type: " + ct)
            cin, cout = _int(l, "channels_in", 1), _int(l, "channels_out", 1)
            if fh == 0 or fw == 0:
                raise ScheduleError("conv layer needs filter_h/filter_w")
            out.schedule.append(Conv(fh, fw, ct == "same", cin, cout))
        elif kind == "activation":
            fn = _str(l, "fn", "identity")
            if fn not in FN:
                raise ScheduleError("unknown activation: " + fn)
            out.schedule.append(Act(FN[fn]))
        else:
            raise ScheduleError('layer kind must be "conv" or "activation"')
    src = doc.get("weights", RANDOM)
    if src not in (RANDOM, FILE):
        raise ScheduleError('weights must be "random" or "file"')
    out.weights_source = src
    mag = doc.get("weight_magnitude", 1)
    if isinstance(mag, bool) or not isinstance(mag, int):
        raise ScheduleError("schedule field 'weight_magnitude' must be an integer")
    if mag < 1:
        raise ScheduleError("weight_magnitude must be >= 1")
    out.weight_magnitude = mag
    return out


def load_schedule_file(path: str) -> ScheduleFile:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ScheduleError("cannot open schedule file: " + path)
    return parse_schedule(text)


def load_integers(path: str) -> np.ndarray:
    """Whitespace-separated integers (REF load_integers)."""
    try:
        with open(path) as f:
            toks = f.read().split()
    except OSError:
        raise ScheduleError("cannot open file: " + path)
    try:
        return np.array([int(t) for t in toks], np.int64)
    except ValueError:
        raise ScheduleError("non-integer content in " + path)


def to_channel_images(values: np.ndarray, channels: int, rows: int, cols: int) -> np.ndarray:
    if values.size != channels * rows * cols:
        raise ScheduleError("image file has wrong element count")
    return values.reshape(channels, rows, cols)


def to_network_weights(values: np.ndarray, schedule) -> List[np.ndarray]:
    """Per conv layer [out][in][fh][fw], consumed in schedule order (REF to_network_weights)."""
    out, idx = [], 0
    for s in schedule:
        if not isinstance(s, Conv):
            continue
        cnt = s.cout * s.cin * s.fh * s.fw
        if idx + cnt > values.size:
            raise ScheduleError("weights file too short for the schedule")
        out.append(values[idx:idx + cnt].reshape(s.cout, s.cin, s.fh, s.fw))
        idx += cnt
    if idx != values.size:
        raise ScheduleError("weights file has trailing values")
    return out


def activation_name(fn: int) -> str:
    return FN_NAME.get(fn, "?")

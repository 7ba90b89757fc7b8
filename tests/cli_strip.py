"""Drop the wall-clock fields from a CLI report so two runs compare equal."""

import csv
import io
import json

CLOCK = ("wall_clock_sec", "total_duration_sec", "first_round_sec", "last_round_sec")


def _drop(obj):
    if isinstance(obj, dict):
        return {k: _drop(v) for k, v in obj.items() if k not in CLOCK}
    if isinstance(obj, list):
        return [_drop(v) for v in obj]
    return obj


def strip_clock(text: str, fmt: str):
    if fmt == "json":
        return _drop(json.loads(text))
    rows = list(csv.DictReader(io.StringIO(text)))
    return [{k: v for k, v in r.items() if k not in CLOCK} for r in rows]

"""JSON documents the CLI writes, validated against the reference's report schemas.

The reference ships JSON-Schema files and validates with ``jsonschema``
(schema.py:14-26, schemas/*.schema.json).  This image has no ``jsonschema``, and
the documents are small and fixed, so the same constraints are restated here as
a few composable checkers; a failure raises ``FormatError`` naming the JSON
pointer of the offending node, as the reference's ``validate_json`` does.
Reports written by either implementation validate under either, which is what
makes a B200 ``bench`` report comparable with a reference one.
"""
from __future__ import annotations

import math
import re

from .errors import FormatError
from .quantize import LAYER_KINDS

_SHA256 = re.compile(r"^[0-9a-f]{64}$")


class _Bad(Exception):
    def __init__(self, path, msg):
        super().__init__(msg)
        self.path, self.msg = path, msg


def _is_int(v):
    return isinstance(v, int) and not isinstance(v, bool)


def _is_num(v):
    return (isinstance(v, (int, float)) and not isinstance(v, bool)
            and not (isinstance(v, float) and not math.isfinite(v)))


def integer(minimum=None, maximum=None):
    def check(v, path):
        if not _is_int(v):
            raise _Bad(path, f"{v!r} is not of type 'integer'")
        if minimum is not None and v < minimum:
            raise _Bad(path, f"{v} is less than the minimum of {minimum}")
        if maximum is not None and v > maximum:
            raise _Bad(path, f"{v} is greater than the maximum of {maximum}")
    return check


def number(minimum=None, nullable=False):
    def check(v, path):
        if v is None and nullable:
            return
        if not _is_num(v):
            raise _Bad(path, f"{v!r} is not of type 'number'")
        if minimum is not None and v < minimum:
            raise _Bad(path, f"{v} is less than the minimum of {minimum}")
    return check


def string(pattern=None):
    def check(v, path):
        if not isinstance(v, str):
            raise _Bad(path, f"{v!r} is not of type 'string'")
        if pattern is not None and not pattern.match(v):
            raise _Bad(path, f"{v!r} does not match {pattern.pattern!r}")
    return check


def one_of(*choices):
    def check(v, path):
        if v not in choices:
            raise _Bad(path, f"{v!r} is not one of {list(choices)}")
    return check


def array(item, min_items=None, max_items=None):
    def check(v, path):
        if not isinstance(v, list):
            raise _Bad(path, f"{v!r} is not of type 'array'")
        if min_items is not None and len(v) < min_items:
            raise _Bad(path, f"{v!r} is too short")
        if max_items is not None and len(v) > max_items:
            raise _Bad(path, f"{v!r} is too long")
        for i, x in enumerate(v):
            item(x, path + [i])
    return check


def obj(required: dict, optional: dict | None = None, values=None):
    """An object with ``required``/``optional`` properties; ``values`` checks the values of
    free-form keys (None = no other keys allowed)."""
    optional = optional or {}

    def check(v, path):
        if not isinstance(v, dict):
            raise _Bad(path, f"{v!r} is not of type 'object'")
        for key in required:
            if key not in v:
                raise _Bad(path, f"{key!r} is a required property")
        for key, x in v.items():
            rule = required.get(key) or optional.get(key)
            if rule is None:
                if values is None:
                    raise _Bad(path, f"additional property {key!r} is not allowed")
                rule = values
            rule(x, path + [key])
    return check


def anything(v, path):
    return None


_TRIPLE = array(integer(1), 3, 3)
_BENCH_CASE = obj(
    {"shape": _TRIPLE, "p": integer(2, 8), "q": integer(2, 8), "group_size": integer(1),
     "stages": integer(1), "workers": integer(1), "wall_ns": integer(0),
     "bmma_passes": integer(0), "effective_GOPS": number(0)},
    {"name": string(), "tile": _TRIPLE})
_KIND = one_of(*LAYER_KINDS)

SCHEMAS = {
    # schemas/bench_report.schema.json
    "bench_report": obj({"suite": string(), "results": array(_BENCH_CASE)}, {"best": _BENCH_CASE}),
    # schemas/manifest.schema.json
    "manifest": obj(
        {"command": string(), "config": obj({}, values=anything),
         "inputs": obj({}, values=string(_SHA256)), "outputs": array(string()),
         "wall_ns": integer(0), "tool_version": string(), "created_at": number()},
        {"stats": obj({}, values=anything)}),
    # schemas/sensitivity_manifest.schema.json
    "sensitivity_manifest": array(obj({"layer_name": string(), "kind": _KIND,
                                       "weight_file": string(), "act_file": string()})),
    # schemas/sensitivity_report.schema.json (sqnr_db / outlier_score null = +inf)
    "sensitivity_report": obj({
        "layers": array(obj({"layer_name": string(), "layer_kind": _KIND,
                             "sqnr_db": number(nullable=True), "output_mse": number(0),
                             "outlier_score": number(1, nullable=True)})),
        "ranking": array(string())}),
}


def validate_json(doc, schema_name: str) -> None:
    """Raise FormatError("invalid <schema> document at /json/pointer: ...") on violation."""
    try:
        SCHEMAS[schema_name](doc, [])
    except _Bad as e:
        pointer = "/" + "/".join(str(p) for p in e.path)
        raise FormatError(f"invalid {schema_name} document at {pointer}: {e.msg}") from None

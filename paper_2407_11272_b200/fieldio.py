"""WVOX1 scalar-field files (SPEC.md:181,
reference winding.py:396-443): one JSON header line, then the raw
little-endian values in flat storage order (k fastest).  The header and
byte layout are identical to the reference's, so files round-trip between
the two packages.  ``gather_and_save`` writes a slab-sharded grid from rank 0.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .errors import ParseError
from .types import GridSpec, ScalarField

__all__ = ["save_field", "load_field", "gather_and_save"]

_CODES = {"f64": "<f8", "f32": "<f4"}


def save_field(field: ScalarField, path) -> None:
    kind = "f32" if np.asarray(field.values).dtype == np.float32 else "f64"
    spec = field.spec
    header = {"magic": "WVOX1", "resolution": list(spec.resolution),
              "bounds_min": [float(x) for x in spec.bounds_min],
              "bounds_max": [float(x) for x in spec.bounds_max],
              "dtype": kind, "order": "zyx-fastest-z"}
    payload = np.ascontiguousarray(field.values, dtype=_CODES[kind]).tobytes()
    with open(path, "wb") as fh:
        fh.write(json.dumps(header).encode("ascii") + b"\n" + payload)


def load_field(path) -> ScalarField:
    name = Path(path).name
    blob = Path(path).read_bytes()
    cut = blob.find(b"\n")
    if cut < 0:
        raise ParseError(f"{name}: missing header line")
    try:
        header = json.loads(blob[:cut].decode("ascii"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise ParseError(f"{name}: bad header: {exc}") from exc
    if not isinstance(header, dict) or header.get("magic") != "WVOX1":
        raise ParseError(f"{name}: not a WVOX1 file")
    try:
        spec = GridSpec(np.array(header["bounds_min"], dtype=np.float64),
                        np.array(header["bounds_max"], dtype=np.float64),
                        tuple(int(r) for r in header["resolution"]))
        code = _CODES[header["dtype"]]
    except (KeyError, TypeError, ValueError) as exc:
        raise ParseError(f"{name}: bad header fields: {exc}") from exc
    values = np.frombuffer(blob[cut + 1:], dtype=code)
    if values.size != spec.num_nodes:
        raise ParseError(f"{name}: expected {spec.num_nodes} values, found {values.size}")
    return ScalarField(spec=spec, values=values.astype(
        np.float64 if header["dtype"] == "f64" else np.float32))


def gather_and_save(driver, spec: GridSpec, path, policy: int = 1) -> None:
    """All-gather a SlabDriver's sharded forward and write it from rank 0."""
    vals, _ = driver.forward(policy=policy, gather=True)
    if driver.rank == 0:
        save_field(ScalarField(spec, vals.detach().cpu().numpy()), path)

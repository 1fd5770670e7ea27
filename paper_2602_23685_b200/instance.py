"""VRP-RPD problem instances: the hot path's input.

Host-side mirror of the reference's ``instance`` module
(``/root/reference/pkg/src/vrp_rpd/instance.py``): the same public names,
argument meanings and error classes, so callers switch by changing the import.
Only the data boundary matters to the device path: ``Instance`` carries
``n``, the (n+1)x(n+1) travel-time matrix ``d`` (depot = location 0), the
processing times ``p`` (``p[0] == 0``) and the fleet ``(m, k)``.  The arrays
are cached as contiguous float64 numpy buffers (``Instance.arrays()``) for
upload by :mod:`paper_2602_23685_b200.device`.

Reference map:
  Instance            instance.py:82-156
  parse_tsplib        instance.py:200-316 (EXPLICIT LOWER_DIAG_ROW/UPPER_ROW/FULL_MATRIX,
                      EUC_2D/CEIL_2D/GEO/ATT)
  fleet_for           instance.py:340-345
  build_instance      instance.py:360-401 (PCG64 SeedSequence streams 17 / 29)
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

VARIANT_KINDS = ("base", "2x", "5x", "1R10", "1R20")
_FIXED_FACTOR = {"base": 1.0, "2x": 2.0, "5x": 5.0}
_RANDOM_CEILING = {"1R10": 10, "1R20": 20}
_STREAM_BASE, _STREAM_MULT = 17, 29


class TsplibParseError(ValueError):
    """Malformed or unsupported TSPLIB text."""


@dataclass(frozen=True)
class RawTsplib:
    name: str
    dimension: int
    edge_weights: np.ndarray

    def __post_init__(self):
        w = self.edge_weights
        if w.shape != (self.dimension, self.dimension):
            raise TsplibParseError(f"matrix shape {w.shape} != dimension {self.dimension}")
        if np.any(np.diag(w) != 0):
            raise TsplibParseError("travel-time matrix has nonzero diagonal entries")
        tol = 1e-9 * max(1.0, float(np.abs(w).max()))
        if float(np.abs(w - w.T).max()) > tol:
            raise TsplibParseError("travel-time matrix is not symmetric")
        if (w < 0).any():
            raise TsplibParseError("negative travel times")


@dataclass(frozen=True)
class VariantSpec:
    kind: str
    seed: int
    replicate: int = 0

    def __post_init__(self):
        if self.kind not in VARIANT_KINDS:
            raise ValueError(f"unknown variant kind {self.kind!r}")


@dataclass(frozen=True)
class FleetConfig:
    m: int
    k: int

    def __post_init__(self):
        if min(self.m, self.k) < 1:
            raise ValueError("fleet requires m >= 1 and k >= 1")


@dataclass(frozen=True)
class Instance:
    """n customers, travel times d (nested tuples, depot 0), processing p."""

    n: int
    d: tuple
    p: tuple
    fleet: FleetConfig
    label: str
    variant: str = "base"
    seed: int = 0
    replicate: int = 0
    _cache: dict = field(default_factory=dict, compare=False, hash=False, repr=False)

    def __post_init__(self):
        if self.n < 1:
            raise ValueError("instance needs at least one customer")
        size = self.n + 1
        if len(self.d) != size or any(len(row) != size for row in self.d):
            raise ValueError("travel-time matrix must be (n+1)x(n+1)")
        if len(self.p) != size or min(self.p) < 0:
            raise ValueError("processing times must cover locations 0..n and be >= 0")

    @property
    def m(self) -> int:
        return self.fleet.m

    @property
    def k(self) -> int:
        return self.fleet.k

    @property
    def customers(self) -> range:
        return range(1, self.n + 1)

    def matrix(self) -> np.ndarray:
        return self.arrays()[0].copy()

    def arrays(self):
        """(d, p) as cached C-contiguous float64 arrays."""
        got = self._cache.get("arrays")
        if got is None:
            d = np.ascontiguousarray(np.array(self.d, dtype=np.float64))
            p = np.ascontiguousarray(np.array(self.p, dtype=np.float64))
            d.setflags(write=False)
            p.setflags(write=False)
            got = self._cache["arrays"] = (d, p)
        return got

    @classmethod
    def from_arrays(cls, d, p, m: int, k: int, label: str = "arrays", **meta) -> "Instance":
        d = np.asarray(d, dtype=np.float64)
        p = np.asarray(p, dtype=np.float64)
        inst = cls(n=d.shape[0] - 1, d=tuple(map(tuple, d.tolist())), p=tuple(p.tolist()),
                   fleet=FleetConfig(int(m), int(k)), label=label, **meta)
        return inst

    def to_dict(self) -> dict:
        return {"label": self.label, "n": self.n, "m": self.m, "k": self.k,
                "matrix": [list(r) for r in self.d], "processing_times": list(self.p[1:]),
                "variant": self.variant, "seed": self.seed, "replicate": self.replicate}

    @classmethod
    def from_dict(cls, doc: dict) -> "Instance":
        return cls(n=int(doc["n"]),
                   d=tuple(tuple(float(x) for x in r) for r in doc["matrix"]),
                   p=(0.0,) + tuple(float(x) for x in doc["processing_times"]),
                   fleet=FleetConfig(int(doc["m"]), int(doc["k"])), label=str(doc["label"]),
                   variant=str(doc.get("variant", "base")), seed=int(doc.get("seed", 0)),
                   replicate=int(doc.get("replicate", 0)))

    def save(self, path) -> None:
        Path(path).write_text(json.dumps(self.to_dict()), encoding="utf-8")

    @classmethod
    def load(cls, path) -> "Instance":
        return cls.from_dict(json.loads(Path(path).read_text(encoding="utf-8")))


# --------------------------------------------------------------------------
# TSPLIB
# --------------------------------------------------------------------------

def _round_half_up(x: float) -> int:  # TSPLIB nint
    return int(x + 0.5)


def _geo_rad(x: float) -> float:
    deg = _round_half_up(x)
    return 3.141592 * (deg + 5.0 * (x - deg) / 3.0) / 180.0


def _pair_distance(kind: str, a, b) -> float:
    dx, dy = a[0] - b[0], a[1] - b[1]
    if kind == "EUC_2D":
        return float(_round_half_up(math.sqrt(dx * dx + dy * dy)))
    if kind == "CEIL_2D":
        return float(math.ceil(math.sqrt(dx * dx + dy * dy)))
    if kind == "ATT":
        r = math.sqrt((dx * dx + dy * dy) / 10.0)
        t = _round_half_up(r)
        return float(t + 1 if t < r else t)
    if kind == "GEO":
        la, oa, lb, ob = _geo_rad(a[0]), _geo_rad(a[1]), _geo_rad(b[0]), _geo_rad(b[1])
        q1, q2, q3 = math.cos(oa - ob), math.cos(la - lb), math.cos(la + lb)
        return float(int(6378.388 * math.acos(0.5 * ((1.0 + q1) * q2 - (1.0 - q1) * q3)) + 1.0))
    raise TsplibParseError(f"unsupported coordinate distance type {kind}")


def _fill_from_explicit(fmt, dim, vals) -> np.ndarray:
    mat = np.zeros((dim, dim))
    if fmt == "FULL_MATRIX":
        want = dim * dim
    elif fmt == "LOWER_DIAG_ROW":
        want = dim * (dim + 1) // 2
    elif fmt == "UPPER_ROW":
        want = dim * (dim - 1) // 2
    else:
        raise TsplibParseError(f"unsupported EDGE_WEIGHT_FORMAT {fmt}")
    if len(vals) != want:
        raise TsplibParseError(f"{fmt} expects {want} entries, found {len(vals)}")
    if fmt == "FULL_MATRIX":
        return np.array(vals, dtype=float).reshape(dim, dim)
    if fmt == "LOWER_DIAG_ROW":
        rows, cols = np.tril_indices(dim)
    else:
        rows, cols = np.triu_indices(dim, 1)
    arr = np.array(vals, dtype=float)
    mat[rows, cols] = arr
    mat[cols, rows] = arr
    return mat


def parse_tsplib(text: str) -> RawTsplib:
    """TSPLIB95 text -> full symmetric matrix (see module docstring)."""
    header: dict = {}
    weights: list = []
    coords: dict = {}
    mode = None
    for raw in text.splitlines():
        line = raw.strip()
        if not line:
            continue
        up = line.upper()
        if up.startswith("EOF"):
            break
        if mode is None and ":" in line:
            key, _, val = line.partition(":")
            header[key.strip().upper()] = val.strip()
            continue
        if up.startswith("EDGE_WEIGHT_SECTION"):
            mode = "w"
        elif up.startswith("NODE_COORD_SECTION"):
            mode = "c"
        elif up.startswith("DISPLAY_DATA_SECTION"):
            mode = "skip"
        elif mode == "w":
            try:
                weights.extend(float(tok) for tok in line.split())
            except ValueError as exc:
                raise TsplibParseError(f"bad token in EDGE_WEIGHT_SECTION: {line!r}") from exc
        elif mode == "c":
            toks = line.split()
            if len(toks) < 3:
                raise TsplibParseError(f"bad node-coordinate line: {line!r}")
            coords[int(float(toks[0]))] = (float(toks[1]), float(toks[2]))
    try:
        dim = int(header["DIMENSION"])
    except (KeyError, ValueError):
        dim = None
    if dim is None or dim < 1:
        raise TsplibParseError("missing or invalid DIMENSION")
    kind = header.get("EDGE_WEIGHT_TYPE")
    if kind is None:
        raise TsplibParseError("missing EDGE_WEIGHT_TYPE")
    kind = kind.upper()
    if kind == "EXPLICIT":
        fmt = header.get("EDGE_WEIGHT_FORMAT", "").upper() or None
        mat = _fill_from_explicit(fmt, dim, weights)
    elif kind in ("EUC_2D", "CEIL_2D", "GEO", "ATT"):
        if len(coords) != dim:
            raise TsplibParseError(f"expected {dim} node coordinates, found {len(coords)}")
        pts = [coords[i] for i in sorted(coords)]
        mat = np.zeros((dim, dim))
        for a in range(dim):
            pa = pts[a]
            for b in range(a + 1, dim):
                mat[a, b] = mat[b, a] = _pair_distance(kind, pa, pts[b])
    else:
        raise TsplibParseError(f"unsupported EDGE_WEIGHT_TYPE {kind}")
    return RawTsplib(name=header.get("NAME") or "unnamed", dimension=dim, edge_weights=mat)


def dump_tsplib(raw: RawTsplib) -> str:
    lines = [f"NAME: {raw.name}", "TYPE: TSP", f"DIMENSION: {raw.dimension}",
             "EDGE_WEIGHT_TYPE: EXPLICIT", "EDGE_WEIGHT_FORMAT: FULL_MATRIX",
             "EDGE_WEIGHT_SECTION"]
    lines += [" " + " ".join(repr(float(x)) for x in row) for row in raw.edge_weights]
    lines.append("EOF")
    return "\n".join(lines) + "\n"


def load_tsplib_file(path) -> RawTsplib:
    return parse_tsplib(Path(path).read_text(encoding="utf-8"))


# --------------------------------------------------------------------------
# Instances
# --------------------------------------------------------------------------

def fleet_for(n: int) -> FleetConfig:
    if n < 1:
        raise ValueError("n must be >= 1")
    return FleetConfig(6, 4) if n >= 24 else FleetConfig(3, 5)


def _pcg(entropy) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy)))


def build_instance(raw: RawTsplib, variant: VariantSpec) -> Instance:
    """Depot = node 0; p = integer base draw over the off-diagonal weight range
    times the variant factor (fixed 1/2/5 or a per-customer U{1..10|20})."""
    if raw.dimension < 2:
        raise ValueError("need at least 2 nodes (depot + 1 customer)")
    n = raw.dimension - 1
    w = raw.edge_weights
    off_diag = w[~np.eye(raw.dimension, dtype=bool)]
    lo_w, hi_w = int(round(float(off_diag.min()))), int(round(float(off_diag.max())))
    base = _pcg([variant.seed, _STREAM_BASE]).integers(lo_w, hi_w + 1, size=n).astype(float)
    if variant.kind in _FIXED_FACTOR:
        p = base * _FIXED_FACTOR[variant.kind]
        label = f"{raw.name}-{variant.kind}-s{variant.seed}"
    else:
        top = _RANDOM_CEILING[variant.kind]
        mult = _pcg([variant.seed, _STREAM_MULT, VARIANT_KINDS.index(variant.kind),
                     variant.replicate]).integers(1, top + 1, size=n)
        p = base * mult
        label = f"{raw.name}-{variant.kind}-s{variant.seed}-r{variant.replicate}"
    return Instance(n=n, d=tuple(map(tuple, w.astype(float).tolist())),
                    p=(0.0,) + tuple(float(x) for x in p), fleet=fleet_for(n), label=label,
                    variant=variant.kind, seed=variant.seed, replicate=variant.replicate)

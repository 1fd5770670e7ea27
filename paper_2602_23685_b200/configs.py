"""The five BASELINE.json configurations as concrete instances.

Only gr17 ships with the reference (``pkg/data/gr17.tsp``); eil51, kroA100,
a280 and dsj1000 are not available offline, so -- as SURVEY.md §8(d) lays
out -- they are synthetic stand-ins with the same node count and TSPLIB
distance type, built through :func:`instance.parse_tsplib` and
:func:`instance.build_instance` with variant seed 136 (the reference's
acceptance seed, ``pkg/tests/test_acceptance.py:35``).  Coordinates are
integer draws from ``numpy.random.default_rng(coord_seed)``, recorded in the
TSPLIB COMMENT line.

gr17 is loaded from ``data/gr17_base.json`` (package data), the reference's own
parse of ``pkg/data/gr17.tsp`` as written by ``tests/golden/make_golden.py``.
"""
from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .instance import Instance, VariantSpec, build_instance, parse_tsplib

VARIANT_SEED = 136
REPO = Path(__file__).resolve().parent.parent
GR17_JSON = Path(__file__).resolve().parent / "data" / "gr17_base.json"


@dataclass(frozen=True)
class ConfigSpec:
    key: str
    nodes: int
    edge_type: str
    span: int
    coord_seed: int
    variant: str
    description: str


CONFIGS = {
    "gr17": ConfigSpec("gr17", 17, "EXPLICIT", 0, 0, "base",
                       "gr17 base: BRKGA population decode + makespan eval"),
    "eil51": ConfigSpec("eil51", 51, "EUC_2D", 70, 5101, "2x",
                        "eil51-derived 2x: ALNS destroy-repair insertion scoring"),
    "kroA100": ConfigSpec("kroA100", 100, "EUC_2D", 4000, 10001, "5x",
                          "kroA100-derived 5x: ALNS->BRKGA warm-start pipeline"),
    "a280": ConfigSpec("a280", 280, "EUC_2D", 300, 28001, "1R10",
                       "a280-derived 1R10: BRKGA island model"),
    "dsj1000": ConfigSpec("dsj1000", 1000, "CEIL_2D", 1_000_000, 100001, "1R20",
                          "dsj1000-derived 1R20: makespan evals/s at n=999"),
}


def synthetic_tsplib(spec: ConfigSpec) -> str:
    rng = np.random.default_rng(spec.coord_seed)
    pts = rng.integers(0, spec.span, size=(spec.nodes, 2))
    lines = [f"NAME: {spec.key}-like",
             f"COMMENT: synthetic stand-in, integer coords U[0,{spec.span}) from "
             f"default_rng({spec.coord_seed})",
             "TYPE: TSP", f"DIMENSION: {spec.nodes}", f"EDGE_WEIGHT_TYPE: {spec.edge_type}",
             "NODE_COORD_SECTION"]
    lines += [f"{i + 1} {int(x)} {int(y)}" for i, (x, y) in enumerate(pts)]
    lines.append("EOF")
    return "\n".join(lines) + "\n"


def config_instance(key: str) -> Instance:
    spec = CONFIGS[key]
    if spec.edge_type == "EXPLICIT":
        if not GR17_JSON.exists():
            raise FileNotFoundError(f"{GR17_JSON} missing (run tests/golden/make_golden.py)")
        return Instance.load(GR17_JSON)
    raw = parse_tsplib(synthetic_tsplib(spec))
    return build_instance(raw, VariantSpec(spec.variant, VARIANT_SEED, 0))

"""Experiment harness (harness.py; the reference's bench.py grid + CSV):
lossless CSV round trip with the reference's field order first (CPU), and a
tiny grid on the GPU whose rows agree with evaluate()."""
import pytest

from paper_2602_23685_b200 import harness as H


def test_rows_csv_round_trip(tmp_path):
    rows = [H.ResultRow("eil51-like", "2x", 0, "budget", 359.0, 20.000123456789, 37.5, 81.25, 42,
                        20.0, 6.02e8, "NVIDIA B200"),
            H.ResultRow("a", "base", 1, "alns", 0.1 + 0.2, 1e-7, 0.0, 100.0, 7)]
    p = tmp_path / "r.csv"
    H.write_rows_csv(rows, p)
    header = p.read_text().splitlines()[0].split(",")
    assert tuple(header[:9]) == H.ResultRow.FIELDS  # the reference's columns, in order
    back = H.read_rows_csv(p)
    key = lambda r: (r.instance, r.variant, r.replicate, r.method)  # noqa: E731
    assert sorted(back, key=key) == sorted(rows, key=key)


@pytest.mark.gpu
def test_tiny_experiment_grid(tmp_path):
    from paper_2602_23685_b200 import alns as A
    from paper_2602_23685_b200 import brkga as B
    from paper_2602_23685_b200.configs import CONFIGS, synthetic_tsplib
    from paper_2602_23685_b200.instance import VariantSpec, build_instance, load_tsplib_file
    from paper_2602_23685_b200.schedule import evaluate
    path = tmp_path / "eil51.tsp"
    path.write_text(synthetic_tsplib(CONFIGS["eil51"]))
    cfg = H.ExperimentConfig([str(path)], kinds=("base", "2x"), replicates={"base": 1, "2x": 1},
                             methods=("alns", "pipeline", "polish", "budget"), seed=3,
                             alns_params=A.AlnsParams(max_iter=20),
                             brkga_params=B.BrkgaParams(population=64, generations=3),
                             budget_s=2.0, out_dir=str(tmp_path / "out"))
    rows, failures = H.run_experiment(cfg)
    assert not failures and len(rows) == 8
    assert (tmp_path / "out" / "results.csv").exists()
    raw = load_tsplib_file(path)
    for r in rows:
        assert r.k1_evals_per_s > 1e6 and r.device
        assert (r.budget_s > 0) == (r.method == "budget")
    by = {(r.variant, r.method): r.makespan for r in rows}
    for kind in ("base", "2x"):
        assert by[(kind, "pipeline")] <= by[(kind, "alns")]  # the better of the two stages
        inst = build_instance(raw, VariantSpec(kind, 3, 0))
        assert by[(kind, "polish")] <= evaluate(inst, A.construct_initial(inst)).makespan

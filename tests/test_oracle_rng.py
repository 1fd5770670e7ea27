"""Oracle RNG + evolve + hint restatement against the reference / numpy."""
import numpy as np
import pytest

import inputs as I
from oracle import oracle as O


def test_evolve_matches_reference(golden, golden_meta):
    for j, ev in enumerate(golden_meta["evolve"]):
        g = I.philox(*ev["pop_key"])
        pop = g.random((ev["N"], ev["G"]))
        fit = g.random(ev["N"])
        if ev["tie"]:
            fit = np.round(fit * 7.0)
        rng = I.philox(*ev["rng_key"])
        out = O.evolve(pop, fit, ev["elite"], ev["mutant"], ev["bias"], rng)
        np.testing.assert_array_equal(out, golden[f"evolve/{j}/out"])
        st = rng.bit_generator.state
        assert [int(x) for x in st["state"]["counter"]] == ev["final_counter"]
        assert int(st["buffer_pos"]) == ev["final_buffer_pos"]
        assert int(st["has_uint32"]) == ev["final_has_uint32"]
        assert int(st["uinteger"]) == ev["final_uinteger"]


def test_hint_vehicle_matches_reference(golden):
    genes = golden["hint/genes"]
    for row, m in zip(golden["hint/out"], (1, 2, 3, 5, 6, 7)):
        assert [O.lib().orc_hint_vehicle(m, float(x)) for x in genes] == list(row)


def test_philox_stream_matches_numpy():
    import ctypes as C
    g = I.philox(136, 7)
    s = O.PhiloxState.from_numpy(g)
    ours = [O.lib().orc_philox_next64(C.byref(s)) for _ in range(13)]
    assert ours == [int(x) for x in I.philox(136, 7).bit_generator.random_raw(13)]


def test_philox_integers_interleaved_with_doubles():
    import ctypes as C
    g = I.philox(1, 2)
    s = O.PhiloxState.from_numpy(g)
    sizes = np.random.default_rng(0).integers(1, 2**32, size=600)
    for i, n in enumerate(sizes):
        if i % 3 == 0:
            assert g.random() == O.lib().orc_philox_next_double(C.byref(s))
        else:
            assert int(g.integers(int(n))) == O.lib().orc_philox_integers(C.byref(s), int(n))


def test_stable_argsort_matches_numpy():
    x = np.random.default_rng(3).random(2001)
    x[::5] = 0.25
    x[7], x[9] = -0.0, 0.0
    np.testing.assert_array_equal(O.stable_argsort(x), np.argsort(x, kind="stable"))


def test_evolve_population_too_small():
    with pytest.raises(ValueError):
        O.evolve(np.zeros((4, 6)), np.arange(4.0), 0.15, 0.15, 0.7, I.philox(0, 0))


@pytest.mark.parametrize("key", [(77, 9), (77, 13), (77, 47)])
def test_forced_rejection_keys_really_reject(key):
    """The keys used by test_gpu_brkga's forced-rejection test do make numpy's
    integers() redraw: with one rejection the Philox stream is one u32 longer
    than the rejection-free count."""
    N, G = 30000, 6
    ne, nm = int(0.15 * N), int(0.15 * N)
    no = N - ne - nm
    g = I.philox(*key)
    g.random((nm, G))
    g.integers(ne, size=no)
    g.integers(N - ne, size=no)
    st = g.bit_generator.state
    consumed_u64 = (int(st["state"]["counter"][0]) - 1) * 4 + int(st["buffer_pos"])
    used32 = 2 * (consumed_u64 - nm * G) - int(st["has_uint32"])
    assert used32 == 2 * no + 1

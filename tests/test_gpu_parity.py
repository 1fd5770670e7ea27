"""GPU parity: the sm_100a kernels (through the C-ABI) against the reference's
golden vectors and the CPU oracle -- bit-exact (integer configs and the
non-integer ones alike, since the kernels keep the reference's fp64 order)."""
import numpy as np
import pytest
import torch

import inputs as I
from conftest import CONFIG_KEYS, config_instance
from oracle import oracle as O

pytestmark = pytest.mark.gpu

CID = {"gr17": 1, "eil51": 2, "kroA100": 3, "a280": 4, "dsj1000": 5}
MODES = ((0, "exact"), (1, "eval"), (2, "two"))


def dev():
    from paper_2602_23685_b200 import device
    return device


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("key", CONFIG_KEYS)
@pytest.mark.parametrize("tag", ["dec", "rnd", "blk", "swp", "mal"])
@pytest.mark.parametrize("op_dtype", [np.int32, np.int16])
def test_makespan_family_vs_golden(key, tag, op_dtype, golden):
    inst = config_instance(key)
    pre = f"{key}/"
    ops = golden[pre + ("dec_ops" if tag == "dec" else f"{tag}_ops")].astype(op_dtype)
    lens = golden[pre + ("dec_lens" if tag in ("dec", "swp") else f"{tag}_lens")]
    for mode, short in MODES:
        if tag == "mal" and mode == 0:
            continue  # exact_makespan does not validate; its result on malformed input is loop-order dependent
        r = dev().makespan_batch(inst, _cuda(ops), _cuda(lens), mode=mode, want_returns=True)
        st = r["status"].cpu().numpy()
        np.testing.assert_array_equal(st, golden[pre + f"{tag}_st_{short}"], err_msg=short)
        np.testing.assert_array_equal(r["z"].cpu().numpy(), golden[pre + f"{tag}_z_{short}"], err_msg=short)
        if mode == 1:
            ok = st == 0
            np.testing.assert_array_equal(r["returns"].cpu().numpy()[ok],
                                          golden[pre + f"{tag}_returns"][ok])


@pytest.mark.parametrize("key", CONFIG_KEYS)
@pytest.mark.parametrize("tag", ["dec", "enc", "strict"])
def test_decode_vs_golden(key, tag, golden):
    inst = config_instance(key)
    pre = f"{key}/"
    n_dec = golden[pre + "dec_ops"].shape[0]
    genes = I.chromosomes(inst.n, n_dec, (136, CID[key]))
    if tag == "enc":
        genes = golden[pre + "enc_genes"]
    elif tag == "strict":
        genes = genes[: golden[pre + "enc_genes"].shape[0]]
    r = dev().decode_batch(inst, _cuda(genes), relax=(tag != "strict"))
    np.testing.assert_array_equal(r["ops"].cpu().numpy(), golden[pre + f"{tag}_ops"])
    np.testing.assert_array_equal(r["lens"].cpu().numpy(), golden[pre + f"{tag}_lens"])
    for f in ("fitness", "makespan", "scheduled", "visits"):
        np.testing.assert_array_equal(r[f].cpu().numpy(), golden[pre + f"{tag}_{f}"], err_msg=f)


@pytest.mark.parametrize("key,count", [("gr17", 4096), ("eil51", 2048), ("kroA100", 1024),
                                       ("a280", 512), ("dsj1000", 256)])
def test_decode_then_score_vs_oracle_at_scale(key, count):
    """Fresh chromosomes (not in the golden set): GPU decode == oracle decode,
    and the decoded makespan equals exact_makespan of the decoded solution
    (SURVEY Appendix A.16 cross-check), int16 and int32 op paths alike."""
    inst = config_instance(key)
    genes = I.chromosomes(inst.n, count, (999, CID[key]))
    g = _cuda(genes)
    r = dev().decode_batch(inst, g)
    ref = O.decode_batch(inst, genes)
    np.testing.assert_array_equal(r["ops"].cpu().numpy(), ref["ops"])
    np.testing.assert_array_equal(r["fitness"].cpu().numpy(), ref["fitness"])
    np.testing.assert_array_equal(r["visits"].cpu().numpy(), ref["visits"])
    r16 = dev().decode_batch(inst, g, op_dtype=torch.int16)
    assert torch.equal(r16["ops"].to(torch.int32), r["ops"])
    for ops in (r["ops"], r16["ops"]):
        s = dev().makespan_batch(inst, ops, r["lens"], mode=0)
        assert (s["status"] == 0).all()
        assert torch.equal(s["z"], r["makespan"])
    z2, st2 = O.makespan_batch(inst, ref["ops"], ref["lens"], mode="two_pass")
    s2 = dev().makespan_batch(inst, r["ops"], r["lens"], mode=2)
    np.testing.assert_array_equal(s2["status"].cpu().numpy(), st2)
    np.testing.assert_array_equal(s2["z"].cpu().numpy(), z2)


@pytest.mark.parametrize("key", ["gr17", "a280"])
def test_evaluate_records_vs_oracle(key, golden):
    inst = config_instance(key)
    ops = golden[f"{key}/dec_ops"][:8]
    lens = golden[f"{key}/dec_lens"][:8]
    r = dev().evaluate_records(inst, _cuda(ops), _cuda(lens))
    for i in range(ops.shape[0]):
        st, z, ret, arr, tim, q0 = O.evaluate_one(inst, ops[i], lens[i])
        assert int(r["status"][i]) == st == 0
        assert float(r["z"][i]) == z
        np.testing.assert_array_equal(r["arrival"][i].cpu().numpy(), arr)
        np.testing.assert_array_equal(r["time"][i].cpu().numpy(), tim)
        np.testing.assert_array_equal(r["q0"][i].cpu().numpy(), q0)


def test_non_integral_instance_bit_exact():
    """fp64 path (no int32 twin): perturbed non-integer d and p."""
    from paper_2602_23685_b200.instance import Instance
    base = config_instance("kroA100")
    d, p = base.arrays()
    rng = np.random.default_rng(5)
    d2 = d + rng.random(d.shape) * 0.37
    d2 = (d2 + d2.T) / 2
    np.fill_diagonal(d2, 0.0)
    p2 = p * 1.0001 + rng.random(p.shape) / 3
    p2[0] = 0.0
    inst = Instance.from_arrays(d2, p2, base.m, base.k, label="kro-frac")
    genes = I.chromosomes(inst.n, 256, (5, 5))
    r = dev().decode_batch(inst, _cuda(genes))
    ref = O.decode_batch(inst, genes)
    np.testing.assert_array_equal(r["ops"].cpu().numpy(), ref["ops"])
    np.testing.assert_array_equal(r["fitness"].cpu().numpy(), ref["fitness"])
    ops, lens = I.random_candidates(inst.n, inst.m, 64, (5, 6))
    ops = np.concatenate([ref["ops"], ops, I.swap_perturb(ref["ops"], ref["lens"], (5, 7))])
    lens = np.concatenate([ref["lens"], lens, ref["lens"]])
    for mode, name in ((0, "exact"), (1, "evaluate"), (2, "two_pass")):
        s = dev().makespan_batch(inst, _cuda(ops), _cuda(lens), mode=mode)
        z, st = O.makespan_batch(inst, ops, lens, mode=name)
        np.testing.assert_array_equal(s["status"].cpu().numpy(), st)
        np.testing.assert_array_equal(s["z"].cpu().numpy(), z)


def test_narrow_ready_overflow_falls_back_exactly():
    """Integral instance whose ready times exceed 32 bits: the narrow K1 pass
    must flag those candidates and the 64-bit fix-up pass reproduce the
    oracle exactly (plus small-time candidates that stay on the narrow path)."""
    from paper_2602_23685_b200.instance import Instance
    base = config_instance("kroA100")
    d, p = base.arrays()
    d2 = np.minimum(d * 100000.0, 2.0**31 - 1)  # integral, < 2^31; route sums pass 2^32
    inst = Instance.from_arrays(d2, p, base.m, base.k, label="kro-huge-d")
    genes = I.chromosomes(inst.n, 512, (17, 17))
    ref = O.decode_batch(inst, genes)
    small = O.decode_batch(base, genes)
    # K3's narrow ready table overflows the same way: its wide fix-up pass must
    # reproduce the oracle decode (int16 and int32 outputs)
    for dt in (torch.int32, torch.int16):
        r = dev().decode_batch(inst, _cuda(genes), op_dtype=dt)
        np.testing.assert_array_equal(r["ops"].cpu().numpy().astype(np.int32), ref["ops"])
        np.testing.assert_array_equal(r["fitness"].cpu().numpy(), ref["fitness"])
        np.testing.assert_array_equal(r["visits"].cpu().numpy(), ref["visits"])
    for mode, name in ((0, "exact"), (1, "evaluate")):
        r = dev().makespan_batch(inst, _cuda(ref["ops"]), _cuda(ref["lens"]), mode=mode)
        z, st = O.makespan_batch(inst, ref["ops"], ref["lens"], mode=name)
        assert (z > 2.0**32).any()
        np.testing.assert_array_equal(r["status"].cpu().numpy(), st)
        np.testing.assert_array_equal(r["z"].cpu().numpy(), z)
        r = dev().makespan_batch(base, _cuda(small["ops"]), _cuda(small["lens"]), mode=mode)
        np.testing.assert_array_equal(r["z"].cpu().numpy(), small["makespan"])


def test_decode_narrow_overflow_at_large_n():
    """n >= 500 decodes through K3's narrow (uint32) ready table; a scaled
    dsj1000 instance pushes some ready times past 2^32, and the wide fix-up
    pass must reproduce the oracle exactly for those and the narrow pass for
    the rest."""
    from paper_2602_23685_b200.instance import Instance
    base = config_instance("dsj1000")
    d, p = base.arrays()
    inst = Instance.from_arrays(d * 5.0, p * 5.0, base.m, base.k, label="dsj-x5")
    genes = I.chromosomes(inst.n, 64, (19, 19))
    ref = O.decode_batch(inst, genes)
    assert (ref["makespan"] > 2.0**32).any() and (ref["makespan"] < 2.0**32).any()
    r = dev().decode_batch(inst, _cuda(genes), op_dtype=torch.int16)
    np.testing.assert_array_equal(r["ops"].cpu().numpy().astype(np.int32), ref["ops"])
    np.testing.assert_array_equal(r["fitness"].cpu().numpy(), ref["fitness"])
    np.testing.assert_array_equal(r["visits"].cpu().numpy(), ref["visits"])


@pytest.mark.parametrize("key", ["eil51", "dsj1000"])
def test_decode_sort_paths_clustered_priorities(key):
    """K3's argsort: uniform priorities take the bucketed counting sort,
    clustered ones (constant, a handful of distinct values, negative / >= 1
    / NaN / -0.0 entries) overflow a bucket and take the bitonic fallback;
    both must give numpy's stable order, hence the oracle's decode."""
    inst = config_instance(key)
    n2 = 2 * inst.n
    g = I.philox(88, 1)
    rows = [np.full(4 * inst.n, 0.5),                                   # one bucket
            np.concatenate([g.integers(0, 4, n2) / 4.0, g.random(n2)]),  # 4 distinct values
            np.concatenate([g.integers(0, 40, n2) / 40.0, g.random(n2)]),  # ~n/20 repeats each
            g.random(4 * inst.n)]                                       # uniform
    odd = g.random(4 * inst.n)
    odd[:8] = [-0.0, 0.0, -1.5, 1.0, 2.0, np.inf, -np.inf, np.nan]
    rows.append(odd)
    genes = np.stack(rows)
    r = dev().decode_batch(inst, _cuda(genes))
    ref = O.decode_batch(inst, genes)
    np.testing.assert_array_equal(r["ops"].cpu().numpy(), ref["ops"])
    np.testing.assert_array_equal(r["fitness"].cpu().numpy(), ref["fitness"])
    np.testing.assert_array_equal(r["visits"].cpu().numpy(), ref["visits"])


def test_decode_narrow_overflow_segmented_kernel():
    """200 <= n < 500 decodes through the segmented K3 kernel (several
    chromosomes per warp) with the narrow ready table: a scaled a280 instance
    pushes about half the chromosomes past 2^32 -- the wide fix-up pass (also
    segmented) must reproduce the oracle for those, the narrow pass for the
    rest."""
    from paper_2602_23685_b200.instance import Instance
    base = config_instance("a280")
    d, p = base.arrays()
    genes = I.chromosomes(base.n, 96, (23, 23))
    z0 = O.decode_batch(base, genes[:16])["makespan"]
    scale = float(np.floor(2.0**32 / np.median(z0)))
    assert d.max() * scale < 2.0**31 and p.max() * scale < 2.0**31
    inst = Instance.from_arrays(d * scale, p * scale, base.m, base.k, label="a280-scaled")
    ref = O.decode_batch(inst, genes)
    assert (ref["makespan"] > 2.0**32).any() and (ref["makespan"] < 2.0**32).any()
    for op_dtype in (torch.int16, torch.int32):
        r = dev().decode_batch(inst, _cuda(genes), op_dtype=op_dtype)
        np.testing.assert_array_equal(r["ops"].cpu().numpy().astype(np.int32), ref["ops"])
        np.testing.assert_array_equal(r["lens"].cpu().numpy(), ref["lens"])
        np.testing.assert_array_equal(r["fitness"].cpu().numpy(), ref["fitness"])
        np.testing.assert_array_equal(r["visits"].cpu().numpy(), ref["visits"])


@pytest.mark.parametrize("key", CONFIG_KEYS)
def test_decode_warp_per_chromosome_kernel(key, golden, monkeypatch):
    """VRP_DECODE_SINGLE=1 forces the warp-per-chromosome K3 kernel (used at
    n >= 500 and m > 16) on every config: same goldens, relaxed and strict."""
    monkeypatch.setenv("VRP_DECODE_SINGLE", "1")
    inst = config_instance(key)
    pre = f"{key}/"
    genes = I.chromosomes(inst.n, golden[pre + "dec_ops"].shape[0], (136, CID[key]))
    for tag, g, relax in (("dec", genes, True), ("strict", genes[: golden[pre + "enc_genes"].shape[0]], False)):
        r = dev().decode_batch(inst, _cuda(g), relax=relax)
        np.testing.assert_array_equal(r["ops"].cpu().numpy(), golden[pre + f"{tag}_ops"])
        for f in ("fitness", "visits"):
            np.testing.assert_array_equal(r[f].cpu().numpy(), golden[pre + f"{tag}_{f}"], err_msg=f)


@pytest.mark.parametrize("key", CONFIG_KEYS)
def test_bottleneck_out_vs_oracle(key, golden):
    """vrp_makespan_batch's bottleneck output = Schedule.bottleneck
    (schedule.py:105-110: the first vehicle with the largest return, strict >)
    on decoded, block and swap-perturbed candidates, exact and evaluate modes."""
    inst = config_instance(key)
    pre = f"{key}/"
    fams = [(golden[pre + "dec_ops"], golden[pre + "dec_lens"]),
            (golden[pre + "blk_ops"], golden[pre + "blk_lens"]),
            (golden[pre + "swp_ops"], golden[pre + "dec_lens"])]
    blk = I.block_candidates(inst.n, inst.m, inst.k, 64, (74, CID[key], 0))
    fams.append(blk)
    for ops, lens in fams:
        for mode, name in ((0, "exact"), (1, "evaluate")):
            r = dev().makespan_batch(inst, _cuda(ops), _cuda(lens), mode=mode, want_returns=True,
                                     want_bottleneck=True)
            z, st, ret = O.makespan_batch(inst, ops, lens, mode=name, want_returns=True)
            ok = st == 0
            assert np.array_equal(r["status"].cpu().numpy(), st)
            want = np.argmax(ret, axis=1)  # first maximum (strict >), like Schedule.bottleneck
            np.testing.assert_array_equal(r["bottleneck"].cpu().numpy()[ok], want[ok], err_msg=name)


@pytest.mark.parametrize("m", [1, 2, 3, 5, 6, 7])
def test_decode_hint_vehicle_edge_values_on_device(m, golden):
    """_hint_vehicle (brkga.py:82-89) on the device at the reference's edge
    values (golden hint/genes: m*g - h within 1e-9 of 1, exact multiples,
    1 - ulp): with capacity for everything every hint vehicle is feasible, so
    the decoded vehicle of each op IS the device's hint; decode must equal the
    oracle's (whose hint is pinned to the reference's goldens)."""
    from paper_2602_23685_b200.instance import Instance
    base = config_instance("gr17")
    d, p = base.arrays()
    inst = Instance.from_arrays(d, p, m, base.n, label=f"gr17-m{m}")
    edge = np.asarray(golden["hint/genes"], dtype=np.float64)
    edge = edge[(edge >= 0.0) & (edge < 1.0)]
    n = inst.n
    rows = 64
    genes = I.chromosomes(n, rows, (93, m))
    hints = np.resize(edge, rows * 2 * n).reshape(rows, 2 * n)
    genes[:, 2 * n:] = hints
    r = dev().decode_batch(inst, _cuda(genes))
    ref = O.decode_batch(inst, genes)
    np.testing.assert_array_equal(r["lens"].cpu().numpy(), ref["lens"])
    np.testing.assert_array_equal(r["ops"].cpu().numpy(), ref["ops"])
    np.testing.assert_array_equal(r["fitness"].cpu().numpy(), ref["fitness"])


def test_max_n_instance_all_scoring_paths():
    """n = VRP_MAX_N = 8192, the largest instance vrp_instance_create accepts:
    K3 decode with uniform priorities (counting sort) and clustered ones (the
    bitonic fallback at its largest shared-memory footprint), then K1 exact /
    evaluate and K2 two-pass on the decoded candidates -- against the oracle."""
    from scipy.spatial.distance import cdist
    from paper_2602_23685_b200.instance import Instance
    n, m, k = 8192, 6, 4
    g = np.random.default_rng(8192)
    xy = g.integers(0, 20000, size=(n + 1, 2)).astype(float)
    d = cdist(xy, xy)
    np.rint(d, out=d)
    p = g.integers(1, 100, size=n + 1).astype(float)
    p[0] = 0
    inst = Instance.from_arrays(d, p, m, k, label="max-n")
    del d
    genes = np.stack([g.random(4 * n),
                      np.concatenate([g.integers(0, 4, 2 * n) / 4.0, g.random(2 * n)])])
    ref = O.decode_batch(inst, genes)
    r = dev().decode_batch(inst, _cuda(genes))
    np.testing.assert_array_equal(r["ops"].cpu().numpy().astype(np.int32), ref["ops"])
    np.testing.assert_array_equal(r["fitness"].cpu().numpy(), ref["fitness"])
    np.testing.assert_array_equal(r["visits"].cpu().numpy(), ref["visits"])
    for mode, name in ((0, "exact"), (1, "evaluate"), (2, "two_pass")):
        rr = dev().makespan_batch(inst, _cuda(ref["ops"]), _cuda(ref["lens"]), mode=mode)
        z, st = O.makespan_batch(inst, ref["ops"], ref["lens"], mode=name)
        np.testing.assert_array_equal(rr["status"].cpu().numpy(), st, err_msg=name)
        np.testing.assert_array_equal(rr["z"].cpu().numpy(), z, err_msg=name)

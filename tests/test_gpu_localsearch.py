"""Device-built local search (localsearch.py, vrp_ls_build + K2/K1) against
the reference's goldens and the host-built neighbourhoods, batched."""
import numpy as np
import pytest
import torch

import inputs as I
from conftest import config_instance
from oracle import oracle as O
import ls_host_ref as H
from paper_2602_23685_b200 import alns as A
from paper_2602_23685_b200 import localsearch as LS
from paper_2602_23685_b200.schedule import Solution, exact_makespan

pytestmark = pytest.mark.gpu
CID = {"gr17": 1, "eil51": 2, "kroA100": 3, "a280": 4, "dsj1000": 5}


@pytest.mark.parametrize("key", ["gr17", "eil51", "kroA100"])
def test_batched_local_search_matches_reference(key, golden):
    inst = config_instance(key)
    ops = golden[f"{key}/dec_ops"][:3]
    lens = golden[f"{key}/dec_lens"][:3]
    for tag, fn in (("pr", LS.pickup_repositioning_batch), ("ca", LS.cross_agent_relocation_batch)):
        o, l, z = fn(inst, ops, lens)
        for j in range(3):
            np.testing.assert_array_equal(l[j].cpu().numpy(), golden[f"ls/{key}/{tag}/{j}/lens"], err_msg=f"{tag} {j}")
            np.testing.assert_array_equal(o[j].cpu().numpy(), golden[f"ls/{key}/{tag}/{j}/ops"], err_msg=f"{tag} {j}")
            assert z[j] == exact_makespan(inst, Solution.from_arrays(o[j].cpu().numpy(), l[j].cpu().numpy()))


@pytest.mark.parametrize("key,count", [("gr17", 24), ("eil51", 16), ("kroA100", 8), ("a280", 3)])
def test_batched_local_search_vs_host_neighbourhoods(key, count):
    """Fresh decoded solutions (several per batch, some already improved by a
    first call) against the host-built variant, both LS kinds."""
    inst = config_instance(key)
    genes = I.chromosomes(inst.n, count, (83, CID[key]))
    dec = O.decode_batch(inst, genes)
    ops, lens = dec["ops"], dec["lens"]
    for kind, fn, host in ((0, LS.pickup_repositioning_batch, H.pickup_repositioning_host),
                           (1, LS.cross_agent_relocation_batch, H.cross_agent_relocation_host)):
        o, l, z = fn(inst, ops, lens)
        o, l = o.cpu().numpy(), l.cpu().numpy()
        for j in range(count):
            ref = host(inst, Solution.from_arrays(ops[j], lens[j]))
            ro, rl = ref.to_arrays(inst.n)
            np.testing.assert_array_equal(l[j], rl, err_msg=f"{kind} {j}")
            np.testing.assert_array_equal(o[j], ro[:2 * inst.n], err_msg=f"{kind} {j}")
            assert z[j] == exact_makespan(inst, ref)


def test_builder_covers_whole_neighbourhood():
    """Every candidate of a small cross neighbourhood is a valid permutation
    of the ops with c's pair on w in (gd < gp) order, each exactly once."""
    inst = config_instance("gr17")
    dec = O.decode_batch(inst, I.chromosomes(inst.n, 1, (5, 5)))
    ops = torch.from_numpy(dec["ops"]).cuda()
    lens = torch.from_numpy(dec["lens"]).cuda()
    o, l = dec["ops"][0], dec["lens"][0]
    c = int(o[0] >> 1) + 1
    pos = np.flatnonzero((o >> 1) + 1 == c)
    ent = []
    cnt = []
    for u in range(inst.m):
        L = int(l[u]) - int(sum(1 for p in pos if sum(l[:u]) <= p < sum(l[:u + 1])))
        ent.append((0, c, u, int(pos[0]), int(pos[1])))
        cnt.append((L + 1) * (L + 2) // 2)
    starts = np.concatenate([[0], np.cumsum(cnt)[:-1]])
    total = int(sum(cnt))
    b_ops, b_lens = LS._build(inst, 1, ops, lens, torch.tensor(ent, dtype=torch.int32).cuda(),
                              torch.from_numpy(starts).cuda(), 0, total, op_dtype=torch.int32)
    b_ops, b_lens = b_ops.cpu().numpy(), b_lens.cpu().numpy()
    seen = set()
    for j in range(total):
        assert sorted(b_ops[j].tolist()) == sorted(o.tolist())
        seen.add(tuple(b_ops[j].tolist()) + tuple(b_lens[j].tolist()))
    assert len(seen) == total

"""Run-to-run and batch-partition determinism on the GPU (the
reference pins bitwise reproducibility across thread counts,
`proj/tests/acceptance.cpp:452-485`).

The fused smoothing step hands lines out by a ticket counter (the CTA -> line
assignment differs between runs) and the cluster kernels exchange carries by
st.async / mbarrier pushes; neither may change a single bit of the result.
The norm reductions use a fixed-order tree, so residual histories are bitwise
too.  Sharding config 3 over ranks means solving a slice of the sections as
its own batch: a section's result must not depend on which batch it is in.
"""
import numpy as np
import pytest

import paper_2507_03812_b200 as pmg

pytestmark = pytest.mark.gpu

SEED = pmg.SEED


def solve_c1(ro):
    geom, prob, grid, st, _ = pmg.baseline_config(1, reference_order=ro)
    s = pmg.MultigridSolver(geom, prob, grid, st)
    s.seeded_rhs(SEED)
    rep = s.solve()
    u = s.solution()
    s.close()
    return u, np.array(rep.residual_norms), rep.iterations


@pytest.mark.parametrize("ro", [True, False], ids=["reforder", "fast"])
def test_c1_run_to_run(ro):
    u1, h1, i1 = solve_c1(ro)
    u2, h2, i2 = solve_c1(ro)
    assert i1 == i2
    assert np.array_equal(u1, u2)
    assert np.array_equal(h1, h2)


def batch(first, count, ro):
    """Sections first..first+count-1 of config 3 as one batched solver."""
    scales = pmg.section_scales(256)[first:first + count]
    geom, prob, grid, st, _ = pmg.baseline_config(3, reference_order=ro)
    s = pmg.MultigridSolver(geom, prob, grid, st, n_sections=count, alpha_scales=scales)
    s.seeded_rhs(SEED + first)  # section i of this batch: mt19937(SEED + first + i)
    s.solve()
    u = s.solution().reshape(count, -1)
    hist = [np.array(r.residual_norms) for r in s.reports]
    its = [r.iterations for r in s.reports]
    s.close()
    return u, hist, its


@pytest.mark.parametrize("ro", [True, False], ids=["reforder", "fast"])
def test_c3_partition_invariance(ro):
    """4 sections as one batch, twice, and as 2 + 2 (the 2-rank shard):
    bitwise equal solutions, histories and iteration counts.  The opt-in fast
    mode is bitwise run to run; across partitions its launch shapes (rows per
    thread of the chunked scans) follow the batch size, so there it is held to
    equal iteration counts and roundoff-level agreement."""
    ua, ha, ia = batch(0, 4, ro)
    ub, hb, ib = batch(0, 4, ro)
    u0, h0, i0 = batch(0, 2, ro)
    u1, h1, i1 = batch(2, 2, ro)
    assert np.array_equal(ua, ub) and ia == ib
    assert all(np.array_equal(x, y) for x, y in zip(ha, hb))
    assert ia == i0 + i1
    if not ro:
        us = np.concatenate([u0, u1])
        assert np.abs(ua - us).max() <= 1e-8 * np.abs(ua).max()
        return
    assert np.array_equal(ua, np.concatenate([u0, u1]))
    assert all(np.array_equal(x, y) for x, y in zip(ha, h0 + h1))


def test_c3_shards_match_one_gpu_batch():
    """1-GPU vs N-GPU sharding: the 256-section batch solved whole, and as the
    eight 32-section slices the ranks of an 8-GPU run own (shard.py), give
    bitwise equal results per section (benched mode)."""
    from paper_2507_03812_b200.shard import section_shard
    u_all, h_all, i_all = batch(0, 256, True)
    for w in (2, 8):
        for r in range(w):
            idx = section_shard(256, r, w)
            if w == 2 and r == 1:
                continue  # the 8-way slices cover the second half again
            u, h, its = batch(idx[0], len(idx), True)
            assert np.array_equal(u, u_all[idx[0]:idx[-1] + 1]), (w, r)
            assert its == i_all[idx[0]:idx[-1] + 1], (w, r)
            assert all(np.array_equal(x, y) for x, y in zip(h, h_all[idx[0]:idx[-1] + 1]))

"""Parity of the CUDA path (through the C ABI) with the CPU oracle.

Bit-exact: in-set masks, counts, iteration counts, per-iteration worklist
statistics, aggregate labels/roots, coarse CSR -- all integer work.
"""
import json
import os
import random

import numpy as np
import pytest

import mis2gen as G
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def M():
    import paper_2204_02934_b200 as m
    return m


def dev(g):
    return (torch.from_numpy(g.rowptr).cuda(), torch.from_numpy(np.ascontiguousarray(g.colinds)).cuda())


def small_graphs(count, seed, nmax=200):
    rng = random.Random(seed)
    out = []
    for k in range(count):
        kind = rng.random()
        n = rng.randrange(0, nmax)
        if kind < 0.6:
            g = G.random_graph(n, rng.choice([0.0, 0.01, 0.03, 0.08, 0.2, 0.3]), seed * 7919 + k,
                               diagonal=rng.random() < 0.5)
        elif kind < 0.8:
            g = G.random_powerlaw_graph(max(n, 2), rng.choice([2, 5, 12]), seed * 7919 + k)
        else:
            g = G.stencil(rng.randrange(1, 9), rng.randrange(1, 9), rng.randrange(1, 5), rng.choice([7, 27]),
                          rng.choice([1, 1, 2, 3]))
        out.append(g)
    return out


def check_mis2(g, seed=0, group=0, scheme="xorstar", stats=False, decide="auto", keys="auto", word_bits=64):
    rp, ci = dev(g)
    r = M().mis2(rp, ci, seed=seed, group=group, scheme=scheme, stats=stats, decide=decide, keys=keys,
                 word_bits=word_bits)
    o = O.mis2(g.rowptr, g.colinds, seed=seed, scheme=scheme, stats=stats, word_bits=word_bits)
    assert np.array_equal(r.in_set.cpu().numpy().astype(bool), o.in_set), g.name
    assert (r.count, r.iterations) == (o.count, o.iterations), g.name
    if stats:
        assert np.array_equal(r.stats, o.stats), (g.name, r.stats, o.stats)
    return r


def test_fig1_replay_gpu():
    """fig:example on the device with the figure's priorities."""
    gold = json.load(open(os.path.join(GOLDEN, "fig1.json")))
    g = G.fig1_graph()
    rp, ci = dev(g)
    prio = torch.tensor(gold["priorities"], dtype=torch.int64)
    r = M().mis2(rp, ci, prio_override=prio)
    assert sorted((np.nonzero(r.in_set.cpu().numpy())[0] + 1).tolist()) == gold["result_1based"]
    assert r.iterations == gold["iterations"]
    r1 = M().mis2(rp, ci, prio_override=prio, max_iters=1, allow_partial=True)
    assert r1.rc == M().ENOTCONVERGED
    assert sorted((np.nonzero(r1.in_set.cpu().numpy())[0] + 1).tolist()) == gold["in_after_iter0"]


@pytest.mark.parametrize("decide", ["pull", "push"])
@pytest.mark.parametrize("chunk", range(6))
def test_random_small_graphs(chunk, decide):
    for g in small_graphs(60, 1000 + chunk):
        check_mis2(g, seed=chunk * 17, decide=decide)


@pytest.mark.parametrize("decide", ["pull", "push", "auto"])
@pytest.mark.parametrize("group", [1, 2, 4, 8, 16, 32])
def test_group_width_invariance(group, decide):
    """§V-D lane grouping never changes results."""
    for g in small_graphs(25, 77, nmax=400) + [G.laplace3d_27pt(20), G.kronecker(11)]:
        check_mis2(g, group=group, decide=decide)


@pytest.mark.parametrize("keys", ["on", "off"])
@pytest.mark.parametrize("decide", ["pull", "push"])
def test_huge_rows_block_path(decide, keys):
    """Rows beyond a warp's share (> 32768 entries) are reduced by the whole
    block (finish_phase): two hubs joined to a sparse random graph."""
    n = 90000
    rng = np.random.default_rng(5)
    e = [(0, j) for j in range(1, 40001)] + [(1, j) for j in range(30000, 75000)]
    e += [tuple(x) for x in rng.integers(2, n, size=(60000, 2)) if x[0] != x[1]]
    g = G.from_edges(n, e)
    check_mis2(g, decide=decide, keys=keys)
    check_mis2(g, decide=decide, keys=keys, seed=3)


@pytest.mark.parametrize("keys", ["on", "off"])
@pytest.mark.parametrize("decide", ["pull", "push"])
def test_column_keys(decide, keys):
    """32-bit column keys (ties in the key class resolved on the full words)
    on random / power-law / stencil graphs, every lane-group width, hub rows;
    the Fixed scheme's and the Fig. 1-like small-id words make ties frequent."""
    gs = small_graphs(40, 4242, nmax=300) + [G.laplace3d_27pt(12), G.kronecker(12),
                                           G.random_powerlaw_graph(4000, 40, 3)]
    for g in gs:
        check_mis2(g, decide=decide, keys=keys)
        check_mis2(g, decide=decide, keys=keys, seed=5, scheme="fixed")
    for grp in (1, 4, 32):
        check_mis2(G.kronecker(11), group=grp, decide=decide, keys=keys)


@pytest.mark.parametrize("decide", ["pull", "push", "auto"])
def test_skewed_graph_paths_forced(decide, monkeypatch):
    """The launch choices run_mis2 makes for skewed graphs (C4), forced on small
    graphs through the library's measurement knobs: rows longer than ONE
    gather batch of their lane group deferred to the block's warps
    (MIS2_HEAVY_BATCHES_RT=1), 32-bit column keys with the one-minimum tie
    path, and the L2 evict_last hint on the key / M-id gathers; MIS-2 and
    Alg. 3 (masked phase-2 call) bit-exact with the oracle."""
    monkeypatch.setenv("MIS2_HEAVY_BATCHES_RT", "1")
    monkeypatch.setenv("MIS2_GATHER_KEEP", "1")
    gs = small_graphs(25, 777, nmax=300) + [G.kronecker(12), G.random_powerlaw_graph(4000, 40, 3),
                                          G.laplace3d_27pt(10), G.elasticity3d(6)]
    for g in gs:
        check_mis2(g, decide=decide, keys="on")
        check_mis2(g, decide=decide, keys="on", seed=7, scheme="fixed")
        check_agg(g, decide=decide, keys="on")
    for grp in (1, 2, 8):
        check_mis2(G.kronecker(11), group=grp, decide=decide, keys="on")
    # the G = 2 small-tile kernel with the global queue of deferred rows
    monkeypatch.setenv("MIS2_SMALL_TILES", "2")
    monkeypatch.setenv("MIS2_GQ_RT", "1")
    for g in [G.kronecker(12), G.kronecker(13), G.random_powerlaw_graph(4000, 40, 3)] + small_graphs(10, 778, 300):
        check_mis2(g, group=2, decide=decide, keys="on")
        check_mis2(g, group=2, decide=decide, keys="off", seed=3)


@pytest.mark.parametrize("decide", ["pull", "push"])
def test_decide_forms_long_rows(decide):
    """Both Decide forms on graphs with rows beyond the deferred-row threshold
    (hubs), with and without a stored diagonal (the push form's IN test)."""
    for g in [G.random_powerlaw_graph(4000, 40, 3), G.kronecker(13), G.random_graph(800, 0.6, 9, diagonal=True),
              G.random_graph(800, 0.6, 9, diagonal=False), G.from_edges(300, [(0, j) for j in range(1, 300)])]:
        check_mis2(g, decide=decide)
        check_mis2(g, decide=decide, seed=99)


@pytest.mark.parametrize("scheme", ["xorstar", "fixed", "xor"])
def test_schemes(scheme):
    for g in [G.grid2d_5pt(10, 10), G.laplace3d_7pt(30), G.elasticity3d(8)]:
        check_mis2(g, scheme=scheme)


@pytest.mark.parametrize("decide", ["pull", "push"])
def test_stats_parity(decide):
    for g in [G.grid2d_5pt(10, 10), G.laplace3d_27pt(30), G.kronecker(12), G.random_graph(300, 0.02, 4)]:
        check_mis2(g, stats=True, decide=decide)


def test_edge_cases():
    for g in [G.from_edges(0, []), G.from_edges(1, []), G.from_edges(37, []), G.from_edges(2, [(0, 1)]),
              G.from_edges(64, [(0, j) for j in range(1, 64)])]:
        check_mis2(g)


def test_config1_full():
    g = G.config_graph(0)
    check_mis2(g, stats=True)
    check_mis2(g, seed=12345)


def test_config2_full():
    """BASELINE.json configs[1]: 27-pt 100^3, the bench workload, default launch."""
    g = G.config_graph(1)
    r = check_mis2(g, stats=True)
    assert (r.count, r.iterations) == (21587, 10)
    check_mis2(g, seed=12345)
    check_mis2(g, decide="push")
    check_mis2(g, decide="pull")


@pytest.mark.slow
def test_config3_full():
    check_mis2(G.config_graph(2))


@pytest.mark.slow
def test_config4_full():
    g = G.config_graph(3)
    check_mis2(g)
    # the instrumented kernel of the skewed launch (no deferred-row queue
    # there: its per-iteration statistics are the paper's structure)
    check_mis2(g, stats=True)


@pytest.mark.slow
def test_config5_mis2_full():
    check_mis2(G.config_graph(4))


def test_determinism_repeat():
    g = G.laplace3d_27pt(60)
    rp, ci = dev(g)
    a = M().mis2(rp, ci).in_set.clone()
    for _ in range(4):
        assert torch.equal(M().mis2(rp, ci).in_set, a)


def test_not_converged():
    g = G.laplace3d_7pt(20)
    rp, ci = dev(g)
    r = M().mis2(rp, ci, max_iters=1, allow_partial=True)
    o = O.mis2(g.rowptr, g.colinds, max_iters=1, allow_partial=True)
    assert r.rc == M().ENOTCONVERGED and r.iterations == 1
    assert np.array_equal(r.in_set.cpu().numpy().astype(bool), o.in_set)
    with pytest.raises(M().Mis2Error):
        M().mis2(rp, ci, max_iters=1)


def test_validate_graph():
    g = G.laplace3d_7pt(6)
    rp, ci = dev(g)
    M().validate_graph(rp, ci)
    bad = ci.clone()
    bad[5] = (bad[5] + 3) % g.n  # breaks symmetry / order
    with pytest.raises(M().Mis2Error) as e:
        M().validate_graph(rp, bad)
    assert e.value.rc == M().EGRAPH
    with pytest.raises(M().Mis2Error):
        M().mis2(rp, bad, validate=True)


def test_mis2_host_e2e():
    g = G.laplace3d_27pt(40)
    rph = torch.from_numpy(g.rowptr).pin_memory()
    cih = torch.from_numpy(g.colinds).pin_memory()
    out = torch.empty(g.n, dtype=torch.uint8).pin_memory()
    cnt, its = M().mis2_host(rph, cih, out)
    o = O.mis2(g.rowptr, g.colinds)
    assert np.array_equal(out.numpy().astype(bool), o.in_set) and (cnt, its) == (o.count, o.iterations)


# ----------------------------------------------------------------- aggregation
def check_agg(g, seed=0, decide="auto", word_bits=64, keys="auto", o=None):
    rp, ci = dev(g)
    a = M().aggregate(rp, ci, seed=seed, decide=decide, word_bits=word_bits, keys=keys)
    if o is None:
        o = O.aggregate(g.rowptr, g.colinds, seed=seed, word_bits=word_bits)
    assert a.num_aggs == o.num_aggs, g.name
    assert np.array_equal(a.labels.cpu().numpy(), o.labels), g.name
    assert np.array_equal(a.roots.cpu().numpy(), o.roots), g.name
    assert a.stats == o.stats, (a.stats, o.stats)
    return a


@pytest.mark.parametrize("decide", ["pull", "push"])
@pytest.mark.parametrize("chunk", range(3))
def test_aggregate_small(chunk, decide):
    """includes the masked phase-2 MIS-2 (reading Q15) under both Decide forms"""
    for g in small_graphs(40, 2000 + chunk):
        check_agg(g, seed=chunk, decide=decide)


def test_aggregate_heavy_leftovers():
    # long rows exercise the block/hash phase-3 path (degree > 512)
    for g in [G.random_powerlaw_graph(3000, 30, 5), G.kronecker(12), G.random_graph(1500, 0.5, 3)]:
        check_agg(g)


def test_aggregate_configs():
    check_agg(G.config_graph(0))
    a = check_agg(G.config_graph(1))
    assert a.num_aggs == 42261


@pytest.mark.slow
def test_aggregate_config3():
    check_agg(G.config_graph(2))


@pytest.mark.slow
def test_aggregate_config4():
    """Alg. 3 on the Kronecker scale-24 graph (configs[3]): labels, roots and
    all 8 statistics bit-exact.  The default launch picks the 32-bit column
    keys for this skewed graph, so the masked phase-2 MIS-2 runs with them."""
    check_agg(G.config_graph(3))


@pytest.mark.parametrize("decide", ["pull", "push"])
def test_aggregate_masked_keys(decide):
    """The masked (phase-2) MIS-2 with the 32-bit column keys forced on:
    small random / power-law / stencil graphs and skewed Kronecker graphs."""
    gs = small_graphs(40, 2500) + [G.kronecker(12), G.random_powerlaw_graph(4000, 20, 3), G.laplace3d_27pt(20)]
    for g in gs:
        check_agg(g, decide=decide, keys="on")
        check_agg(g, seed=5, decide=decide, keys="on")


# ----------------------------------------------------------------- coarsening
def check_coarsen(g, labels=None, na=None):
    rp, ci = dev(g)
    if labels is None:
        o = O.aggregate(g.rowptr, g.colinds)
        labels, na = o.labels, o.num_aggs
    crow, ccol = M().coarsen(rp, ci, torch.from_numpy(labels).cuda(), na)
    orow, ocol = O.coarsen(g.rowptr, g.colinds, labels, na)
    assert np.array_equal(crow.cpu().numpy(), orow) and np.array_equal(ccol.cpu().numpy(), ocol), g.name


def test_coarsen_small():
    for g in small_graphs(30, 3000):
        if g.n:
            check_coarsen(g)


def test_coarsen_segments_all_paths():
    g = G.random_graph(2000, 0.3, 9)  # big segments -> block + bitmap paths
    rng = np.random.default_rng(0)
    for na in (1, 3, 40, 700):
        labels = rng.integers(0, na, g.n).astype(np.int32)
        labels[:na] = np.arange(na)
        check_coarsen(g, labels, na)
    check_coarsen(G.config_graph(1))


def test_coarsen_capacity_two_call():
    g = G.laplace3d_7pt(10)
    o = O.aggregate(g.rowptr, g.colinds)
    rp, ci = dev(g)
    import ctypes
    m = M()
    gg, n, nnz = m._graph(rp, ci)
    ws, wsb = m.workspace(m.OP_COARSEN, n, nnz)
    lab = torch.from_numpy(o.labels).cuda()
    crow = torch.empty(o.num_aggs + 1, dtype=torch.int64, device="cuda")
    c = ctypes.c_int64(0)
    small = torch.empty(4, dtype=torch.int32, device="cuda")
    rc = m.lib().mis2_coarsen(ctypes.byref(gg), lab.data_ptr(), o.num_aggs, crow.data_ptr(), small.data_ptr(), 4,
                              ctypes.byref(c), ws.data_ptr(), wsb, m._stream())
    assert rc == m.ERANGE and c.value == len(O.coarsen(g.rowptr, g.colinds, o.labels, o.num_aggs)[1])


def test_multilevel_elasticity():
    g = G.elasticity3d(30)
    rp, ci = dev(g)
    levels, (frp, fci), _ = M().multilevel(rp, ci, threshold=1000)
    olevels, (orp, oci) = O.multilevel(g.rowptr, g.colinds, threshold=1000)
    assert levels == olevels
    assert np.array_equal(frp.cpu().numpy(), orp) and np.array_equal(fci.cpu().numpy(), oci)


@pytest.mark.slow
def test_multilevel_config5():
    """configs[4] (3-dof 27-pt 150^3): level-0 labels, roots, statistics and
    coarse CSR element-wise against the oracle, then every level size and
    the final coarse CSR of the multilevel run."""
    g = G.config_graph(4)
    oa = O.aggregate(g.rowptr, g.colinds)
    a = check_agg(g, o=oa)
    rp, ci = dev(g)
    crow, ccol = M().coarsen(rp, ci, a.labels, a.num_aggs)
    orow, ocol = O.coarsen(g.rowptr, g.colinds, oa.labels, oa.num_aggs)
    assert np.array_equal(crow.cpu().numpy(), orow) and np.array_equal(ccol.cpu().numpy(), ocol)
    levels, (frp, fci), _ = M().multilevel(rp, ci, threshold=1000)
    olevels_rest, (orp, oci) = O.multilevel(orow, ocol, threshold=1000)
    assert levels == [(g.n, int(g.rowptr[-1]), oa.num_aggs)] + olevels_rest
    assert np.array_equal(frp.cpu().numpy(), orp) and np.array_equal(fci.cpu().numpy(), oci)


# ----------------------------------------------------------------- Alg. 2 (NEXT-1)
@pytest.mark.parametrize("chunk", range(2))
def test_basic_coarsening_alg2(chunk):
    gs = small_graphs(30, 4000 + chunk) + [G.config_graph(0), G.laplace3d_27pt(30), G.kronecker(11)]
    for g in gs:
        rp, ci = dev(g)
        a = M().aggregate(rp, ci, basic=True, seed=chunk)
        labels, na = O.coarsen_basic(g.rowptr, g.colinds, seed=chunk)
        assert a.num_aggs == na and np.array_equal(a.labels.cpu().numpy(), labels), g.name


# ----------------------------------------------------------------- partitioned (§8(e))
@pytest.mark.parametrize("nparts", [1, 2, 3, 4, 8])
def test_partitioned_local_transport(nparts):
    """The multi-GPU driver with P partitions on this GPU (halo copies in
    device memory): bit-identical to one GPU and to the oracle."""
    gs = [G.config_graph(0), G.laplace3d_27pt(30), G.kronecker(11), G.random_graph(500, 0.02, 8),
          G.elasticity3d(6), G.random_powerlaw_graph(2000, 6, 4), G.from_edges(5, [])]
    for g in gs:
        for seed in (0, 99):
            c = M().Comm.local_parts(nparts).set_graph(g.n, g.rowptr, g.colinds)
            out = torch.empty(max(g.n, 1), dtype=torch.uint8, device="cuda")
            cnt, its = c.mis2(out, seed=seed)
            c.close()
            o = O.mis2(g.rowptr, g.colinds, seed=seed)
            assert np.array_equal(out[: g.n].cpu().numpy().astype(bool), o.in_set), (g.name, nparts)
            assert (cnt, its) == (o.count, o.iterations), (g.name, nparts)


def test_partitioned_config2_8parts():
    g = G.config_graph(1)
    c = M().Comm.local_parts(8).set_graph(g.n, g.rowptr, g.colinds)
    out = torch.empty(g.n, dtype=torch.uint8, device="cuda")
    cnt, its = c.mis2(out)
    rp, ci = dev(g)
    r = M().mis2(rp, ci)
    assert torch.equal(out, r.in_set) and (cnt, its) == (r.count, r.iterations)


@pytest.mark.parametrize("nparts", [1, 2, 3, 5, 8])
def test_partitioned_aggregate_local_transport(nparts):
    """Alg. 3 over P partitions (mis2_dist_aggregate, halo exchanges of root
    ids / labels, global root numbering, summed aggregate sizes): labels,
    count and all statistics bit-identical to the oracle."""
    gs = [G.config_graph(0), G.laplace3d_27pt(16), G.kronecker(11), G.random_graph(600, 0.02, 8),
          G.elasticity3d(5), G.random_powerlaw_graph(3000, 30, 5), G.from_edges(5, [])]
    for g in gs:
        for seed in (0, 7):
            c = M().Comm.local_parts(nparts).set_graph(g.n, g.rowptr, g.colinds)
            lab = torch.empty(max(g.n, 1), dtype=torch.int32, device="cuda")
            na, st = c.aggregate(lab, seed=seed)
            c.close()
            o = O.aggregate(g.rowptr, g.colinds, seed=seed)
            assert na == o.num_aggs, (g.name, nparts)
            assert np.array_equal(lab[: g.n].cpu().numpy(), o.labels), (g.name, nparts)
            assert st == o.stats, (g.name, nparts, st, o.stats)


def test_partitioned_aggregate_config2_8parts():
    g = G.config_graph(1)
    c = M().Comm.local_parts(8).set_graph(g.n, g.rowptr, g.colinds)
    lab = torch.empty(g.n, dtype=torch.int32, device="cuda")
    na, st = c.aggregate(lab)
    rp, ci = dev(g)
    a = M().aggregate(rp, ci)
    assert na == a.num_aggs and torch.equal(lab, a.labels) and st == a.stats


@pytest.mark.parametrize("nparts", [1, 2, 3, 8])
def test_partitioned_coarsen_and_multilevel(nparts):
    """mis2_dist_coarsen (per-part coarse rows, stacked and merged) equals
    mis2_coarsen / the oracle; the partitioned multilevel equals the
    single-GPU one level by level (NEXT-3)."""
    for g in [G.config_graph(0), G.laplace3d_27pt(14), G.elasticity3d(7), G.random_graph(400, 0.03, 2),
              G.kronecker(10)]:
        c = M().Comm.local_parts(nparts).set_graph(g.n, g.rowptr, g.colinds)
        lab = torch.empty(max(g.n, 1), dtype=torch.int32, device="cuda")
        na, _ = c.aggregate(lab)
        crow, ccol = c.coarsen(lab, na)
        oa = O.aggregate(g.rowptr, g.colinds)
        orow, ocol = O.coarsen(g.rowptr, g.colinds, oa.labels, oa.num_aggs)
        assert np.array_equal(crow.cpu().numpy(), orow) and np.array_equal(ccol.cpu().numpy(), ocol), (g.name, nparts)
        rp, ci = dev(g)
        lv1, fin1, _ = M().multilevel(rp, ci, threshold=50)
        lv, fin = c.multilevel(lab, threshold=50)
        c.close()
        assert [l[0] for l in lv] == [l[0] for l in lv1] and [l[2] for l in lv] == [l[2] for l in lv1], g.name
        if fin is not None:
            assert torch.equal(fin[0], fin1[0]) and torch.equal(fin[1], fin1[1])


@pytest.mark.slow
def test_partitioned_aggregate_config3():
    """configs[3]'s workload: Alg. 3 of the 7-pt 300^3 graph row-partitioned
    over 2, 4 and 8 parts (local transport) -- labels and statistics
    bit-exact against the oracle."""
    g = G.config_graph(2)
    o = O.aggregate(g.rowptr, g.colinds)
    lab = torch.empty(g.n, dtype=torch.int32, device="cuda")
    for nparts in (2, 4, 8):
        c = M().Comm.local_parts(nparts).set_graph(g.n, g.rowptr, g.colinds)
        na, st = c.aggregate(lab)
        c.close()
        assert na == o.num_aggs and st == o.stats, nparts
        assert np.array_equal(lab.cpu().numpy(), o.labels), nparts


@pytest.mark.slow
def test_partitioned_config3_4parts():
    g = G.config_graph(2)
    c = M().Comm.local_parts(4).set_graph(g.n, g.rowptr, g.colinds)
    out = torch.empty(g.n, dtype=torch.uint8, device="cuda")
    cnt, its = c.mis2(out)
    o = O.mis2(g.rowptr, g.colinds)
    assert np.array_equal(out.cpu().numpy().astype(bool), o.in_set) and (cnt, its) == (o.count, o.iterations)


def test_coarsen_bitmap_path():
    # one aggregate with > 2048 distinct neighbour labels forces the bitmap path
    g = G.random_graph(6000, 0.01, 21)
    rng = np.random.default_rng(1)
    na = 3000
    labels = rng.integers(0, na, g.n).astype(np.int32)
    labels[:na] = np.arange(na)
    labels[na: na + 2500] = 7  # aggregate 7 gets ~2500 members x ~60 neighbours
    check_coarsen(g, labels, na)


# ------------------------------------------------------------------ Alg. 4
def cgs_graphs():
    return [G.grid2d_5pt(10, 10), G.laplace3d_7pt(9), G.laplace3d_27pt(8), G.random_graph(300, 0.03, 5),
            G.random_powerlaw_graph(800, 8, 3), G.elasticity3d(4), G.kronecker(9)]


@pytest.mark.parametrize("seed", [0, 17])
def test_coloring_gpu(seed):
    """mis2_color == the oracle's greedy colouring (reading Q30), bit-exact."""
    for g in cgs_graphs() + [G.from_edges(20, []), G.from_edges(0, [])]:
        rp, ci = dev(g)
        c, nc = M().color(rp, ci, seed=seed)
        oc, onc = O.color_jp(g.rowptr, g.colinds, seed=seed)
        assert nc == onc and np.array_equal(c.cpu().numpy(), oc), g.name


@pytest.mark.parametrize("point", [False, True])
def test_cluster_sgs_gpu(point):
    """Alg. 4 sweeps on the GPU == the oracle (fp64; only the order of the
    row sums differs: relative 1e-12), forward / backward / symmetric,
    several sweeps, point and MIS-2-aggregate clusters."""
    rng = np.random.default_rng(11)
    for g0 in cgs_graphs():
        g, vals = G.spd_values(g0, seed=3)
        rp, ci = dev(g)
        vd = torch.from_numpy(vals).cuda()
        if point:
            cg = M().ClusterSGS(rp, ci, vd)
            labels, na, ccolor, nc = O.cgs_setup(g.rowptr, g.colinds, point=True)
        else:
            a = M().aggregate(rp, ci)
            cg = M().ClusterSGS(rp, ci, vd, labels=a.labels, num_aggs=a.num_aggs)
            labels, na, ccolor, nc = O.cgs_setup(g.rowptr, g.colinds)
            assert a.num_aggs == na
        assert cg.ncolors == nc, g.name
        b = rng.standard_normal(g.n)
        x0 = rng.standard_normal(g.n)
        for direction, sweeps in (("forward", 1), ("backward", 1), ("symmetric", 3)):
            x = torch.from_numpy(x0.copy()).cuda()
            cg.apply(torch.from_numpy(b).cuda(), x, sweeps=sweeps, direction=direction)
            want = O.cluster_sgs(g.rowptr, g.colinds, vals, labels, na, ccolor, nc, b, x0, sweeps, direction)
            got = x.cpu().numpy()
            assert np.allclose(got, want, rtol=1e-12, atol=1e-12 * np.abs(want).max()), (g.name, direction)
        cg.close()


@pytest.mark.parametrize("size", [5, 32, 33, 64, 65, 90])
def test_cluster_sgs_given_clusters(size):
    """Clusters given by the caller: rows in blocks of `size` (clusters of
    up to 90 rows, rows of a cluster adjacent to each other), against the
    oracle with the same clusters and the oracle's colouring of the oracle's
    coarse graph."""
    rng = np.random.default_rng(size)
    for g0 in [G.laplace3d_27pt(7), G.grid2d_5pt(20, 13), G.random_graph(400, 0.02, 9)]:
        g, vals = G.spd_values(g0, seed=5)
        labels = (np.arange(g.n) // size).astype(np.int32)
        na = int(labels.max()) + 1
        crow, ccol = O.coarsen(g.rowptr, g.colinds, labels, na)
        ccolor, nc = O.color_jp(crow, ccol)
        rp, ci = dev(g)
        coarse = (torch.from_numpy(np.asarray(crow, dtype=np.int64)).cuda(),
                  torch.from_numpy(np.asarray(ccol, dtype=np.int32)).cuda())
        cg = M().ClusterSGS(rp, ci, torch.from_numpy(vals).cuda(), labels=torch.from_numpy(labels).cuda(),
                            num_aggs=na, coarse=coarse)
        assert cg.ncolors == nc
        b = rng.standard_normal(g.n)
        x0 = rng.standard_normal(g.n)
        for direction in ("forward", "backward", "symmetric"):
            x = torch.from_numpy(x0.copy()).cuda()
            cg.apply(torch.from_numpy(b).cuda(), x, sweeps=2, direction=direction)
            want = O.cluster_sgs(g.rowptr, g.colinds, vals, labels, na, ccolor, nc, b, x0, 2, direction)
            assert np.allclose(x.cpu().numpy(), want, rtol=1e-12, atol=1e-12 * np.abs(want).max()), (g.name, direction)
        cg.close()


def test_cluster_sgs_errors():
    g = G.grid2d_5pt(4, 4)  # no stored diagonal values -> A_ii missing
    rp, ci = dev(G.strip_diagonal(g))
    vals = torch.ones(int(ci.numel()), dtype=torch.float64, device="cuda")
    with pytest.raises(M().Mis2Error):
        M().ClusterSGS(rp, ci, vals)


# ----------------------------------------------------------------- W = 32 status words (§8 f2)
@pytest.mark.parametrize("decide", ["pull", "push"])
@pytest.mark.parametrize("chunk", range(2))
def test_word32_small_graphs(chunk, decide):
    """MIS2_FLAG_WORD32 (reading Q32): bit-exact with the oracle's
    32-bit words, every scheme, both Decide forms."""
    for k, g in enumerate(small_graphs(30, 5000 + chunk)):
        check_mis2(g, seed=k, scheme=("xorstar", "fixed", "xor")[k % 3], decide=decide, word_bits=32, stats=True)


@pytest.mark.parametrize("keys", ["auto", "on"])
def test_word32_structured_and_config2(keys):
    for g in [G.laplace3d_7pt(30), G.elasticity3d(8), G.kronecker(12), G.random_powerlaw_graph(3000, 30, 5)]:
        check_mis2(g, keys=keys, word_bits=32)
    check_mis2(G.config_graph(1), keys=keys, word_bits=32)


def test_word32_aggregate_and_partitioned():
    for g in small_graphs(15, 5100) + [G.laplace3d_27pt(16), G.kronecker(11)]:
        check_agg(g, word_bits=32)
    for g in [G.laplace3d_27pt(16), G.random_powerlaw_graph(2000, 6, 4)]:
        for nparts in (2, 5):
            c = M().Comm.local_parts(nparts).set_graph(g.n, g.rowptr, g.colinds)
            out = torch.empty(max(g.n, 1), dtype=torch.uint8, device="cuda")
            cnt, its = c.mis2(out, word_bits=32)
            lab = torch.empty(max(g.n, 1), dtype=torch.int32, device="cuda")
            na, st = c.aggregate(lab, word_bits=32)
            c.close()
            o = O.mis2(g.rowptr, g.colinds, word_bits=32)
            assert np.array_equal(out[: g.n].cpu().numpy().astype(bool), o.in_set) and (cnt, its) == (o.count, o.iterations)
            oa = O.aggregate(g.rowptr, g.colinds, word_bits=32)
            assert na == oa.num_aggs and np.array_equal(lab[: g.n].cpu().numpy(), oa.labels) and st == oa.stats


# ----------------------------------------------------------------- boundary (include/mis2.h)
def test_int32_rowptr():
    """rowptr_bits = 32: int32 row pointers give the same MIS-2, aggregation,
    coarse graph and validation as int64 ones."""
    for g in [G.config_graph(0), G.laplace3d_27pt(20), G.kronecker(10), G.random_graph(300, 0.05, 1)]:
        rp, ci = dev(g)
        rp32 = rp.to(torch.int32)
        r64, r32 = M().mis2(rp, ci), M().mis2(rp32, ci)
        assert torch.equal(r64.in_set, r32.in_set) and (r64.count, r64.iterations) == (r32.count, r32.iterations)
        a64, a32 = M().aggregate(rp, ci), M().aggregate(rp32, ci)
        assert torch.equal(a64.labels, a32.labels) and a64.stats == a32.stats
        c64, c32 = M().coarsen(rp, ci, a64.labels, a64.num_aggs), M().coarsen(rp32, ci, a64.labels, a64.num_aggs)
        assert torch.equal(c64[0], c32[0]) and torch.equal(c64[1], c32[1])
        M().validate_graph(rp32, ci)
        o = O.mis2(g.rowptr, g.colinds)
        assert np.array_equal(r32.in_set.cpu().numpy().astype(bool), o.in_set)


def test_validate_malformed_rowptr():
    """A malformed rowptr is EGRAPH (not a device fault): the symmetry pass
    only runs on a sound rowptr."""
    g = G.laplace3d_7pt(8)
    rp, ci = dev(g)
    for bad in ([(3, -5)], [(4, g.rowptr[-1] * 4)], [(5, 2), (6, 1)], [(g.n, g.rowptr[-1] + 7)]):
        b = rp.clone()
        for i, v in bad:
            b[i] = int(v)
        with pytest.raises(M().Mis2Error) as e:
            M().validate_graph(b, ci)
        assert e.value.rc == M().EGRAPH
    r = M().mis2(rp, ci)  # the context is still usable
    assert r.count == O.mis2(g.rowptr, g.colinds).count


def test_coarsen_labels_out_of_range():
    """Labels outside [0, num_aggs) are rejected with EINVAL before any kernel
    indexes with them; the device context stays usable."""
    g = G.laplace3d_7pt(10)
    rp, ci = dev(g)
    a = M().aggregate(rp, ci)
    for bad_val in (-7, a.num_aggs, 1 << 30):
        lab = a.labels.clone()
        lab[17] = bad_val
        with pytest.raises(M().Mis2Error) as e:
            M().coarsen(rp, ci, lab, a.num_aggs)
        assert e.value.rc == M().EINVAL
    torch.cuda.synchronize()
    check_coarsen(g)


def test_empty_graph_null_rowptr():
    """n = 0 with NULL rowptr / colinds: empty set, 0 iterations, no kernel."""
    import ctypes
    m = M()
    g = m._Graph(0, 0, None, None, 64, 0)
    o = m._opts()
    ws, wsb = m.workspace(m.OP_MIS2, 0, 0)
    cnt, its = ctypes.c_int64(-1), ctypes.c_int32(-1)
    out = torch.empty(1, dtype=torch.uint8, device="cuda")
    rc = m.lib().mis2(ctypes.byref(g), ctypes.byref(o), out.data_ptr(), ctypes.byref(cnt), ctypes.byref(its), None,
                      ws.data_ptr(), wsb, m._stream())
    assert rc == 0 and cnt.value == 0 and its.value == 0
    torch.cuda.synchronize()


def test_nccl_transport_world1():
    """The NCCL transport (one process per GPU) on the single GPU of this box,
    world size 1: ncclCommInitRank, the request-count allgather of
    set_graph, the per-iteration allreduce of |worklist_1|, the root-count
    allgather of the aggregation and the coarse-CSR allgather of
    mis2_dist_coarsen all run; results bit-identical to the oracle."""
    m = M()
    for g in [G.config_graph(0), G.laplace3d_27pt(20), G.kronecker(10)]:
        c = m.Comm.nccl(m.comm_unique_id(), 1, 0).set_graph(g.n, g.rowptr, g.colinds)
        out = torch.empty(g.n, dtype=torch.uint8, device="cuda")
        cnt, its = c.mis2(out)
        o = O.mis2(g.rowptr, g.colinds)
        assert np.array_equal(out.cpu().numpy().astype(bool), o.in_set) and (cnt, its) == (o.count, o.iterations)
        lab = torch.empty(g.n, dtype=torch.int32, device="cuda")
        na, st = c.aggregate(lab)
        oa = O.aggregate(g.rowptr, g.colinds)
        assert na == oa.num_aggs and st == oa.stats and np.array_equal(lab.cpu().numpy(), oa.labels)
        crow, ccol = c.coarsen(lab, na)
        orow, ocol = O.coarsen(g.rowptr, g.colinds, oa.labels, oa.num_aggs)
        assert np.array_equal(crow.cpu().numpy(), orow) and np.array_equal(ccol.cpu().numpy(), ocol)
        c.close()


@pytest.mark.parametrize("sub", ["0", "1"])
def test_aggregate_phase2_forms(sub, monkeypatch):
    """Phase 2's MIS-2 as the masked call on G and on the induced subgraph of
    the unaggregated vertices (row = vertex gid[row], original ids in the
    hash and the packing): identical labels, roots and statistics."""
    monkeypatch.setenv("MIS2_AGG_SUB", sub)
    gs = small_graphs(30, 2700) + [G.laplace3d_7pt(20), G.kronecker(11), G.elasticity3d(6), G.config_graph(1)]
    for g in gs:
        check_agg(g)
        check_agg(g, seed=3, decide="push")


def test_aggregate_graph_replay():
    """Repeated mis2_aggregate() calls on the same buffers: the first runs
    directly, the second captures the launch sequence into a CUDA graph, the
    later ones replay it -- every result equals the oracle's, also after the
    buffers are refilled with another graph of the same size (a replay reads
    the current contents)."""
    import ctypes
    m = M()
    g1 = G.laplace3d_27pt(14)
    # a second graph with exactly g1's n and nnz: g1 with its ids permuted
    perm = np.random.RandomState(3).permutation(g1.n)
    inv = np.argsort(perm)
    rows = [np.sort(perm[g1.colinds[g1.rowptr[inv[v]]:g1.rowptr[inv[v] + 1]]]) for v in range(g1.n)]
    rp2 = np.zeros(g1.n + 1, dtype=np.int64)
    rp2[1:] = np.cumsum([len(r) for r in rows])
    ci2 = np.concatenate(rows).astype(np.int32)
    rp, ci = dev(g1)
    gg, n, nnz = m._graph(rp, ci)
    o = m._opts(0, "xorstar", 0, 0)
    ws, wsb = m.workspace(m.OP_AGGREGATE, n, nnz)
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    roots = torch.empty(n, dtype=torch.int32, device="cuda")
    na = ctypes.c_int64(0)
    st = np.zeros(8, dtype=np.int64)

    def call_and_check(rowptr, colinds):
        rc = m.lib().mis2_aggregate(ctypes.byref(gg), ctypes.byref(o), labels.data_ptr(), ctypes.byref(na),
                                    roots.data_ptr(), st.ctypes.data, ws.data_ptr(), wsb, m._stream())
        assert rc == 0
        ref = O.aggregate(rowptr, colinds)
        assert na.value == ref.num_aggs
        assert np.array_equal(labels.cpu().numpy(), ref.labels)
        assert np.array_equal(roots.cpu().numpy()[:ref.num_aggs], ref.roots[:ref.num_aggs])

    for _ in range(3):
        call_and_check(g1.rowptr, g1.colinds)
    rp.copy_(torch.from_numpy(rp2))
    ci.copy_(torch.from_numpy(ci2))
    for _ in range(2):
        call_and_check(rp2, ci2)

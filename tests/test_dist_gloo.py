"""Multi-process (gloo, CPU) test of the partitioned MIS-2 protocol.

Each rank plans its row slice with the library's host planner
(``mis2_plan_part`` of libmis2.so -- the same code the GPU driver uses),
exchanges its ghost request lists, and then runs Alg. 1 on its rows with the
exact exchange schedule of csrc/dist.cu: ghost T before every Refresh Column,
ghost M before every Decide, |worklist_1| summed after every Decide.  The
gathered in-set and iteration count must equal the CPU oracle (SURVEY.md P13:
partitioned oracle == monolithic oracle)."""
import os
import socket

import numpy as np
import pytest

import mis2gen as G
import oracle as O

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graphs():
    return {"c1": G.grid2d_5pt(10, 10), "lap": G.laplace3d_27pt(9, 7, 6), "er": G.random_graph(150, 0.04, 3),
            "kron": G.kronecker(9), "elast": G.elasticity3d(4, 3, 3)}


def _rank_main(rank, world, port, name, seed, outdir):
    import torch.distributed as dist

    import paper_2204_02934_b200 as m
    import pins

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = _graphs()[name]
    n = g.n
    lo, hi = n * rank // world, n * (rank + 1) // world
    n_own = hi - lo
    ghosts, req, loc = m.plan_part(n, world, rank, g.rowptr[lo:hi + 1], g.colinds)
    recv_off = np.concatenate([[0], np.cumsum(req)])
    mine = [ghosts[recv_off[q]:recv_off[q + 1]] for q in range(world)]
    allreq = [None] * world
    dist.all_gather_object(allreq, mine)
    send_idx = {p: np.asarray(allreq[p][rank], dtype=np.int64) - lo for p in range(world) if p != rank}
    nt = n_own + len(ghosts)
    # closed neighbourhoods of the owned rows in the local index space
    rp = g.rowptr[lo:hi + 1] - g.rowptr[lo]
    rows = np.repeat(np.arange(n_own), np.diff(rp))
    rows = np.concatenate([rows, np.arange(n_own)])
    cols = np.concatenate([loc.astype(np.int64), np.arange(n_own)])
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    starts = np.searchsorted(rows, np.arange(n_own))
    OUT = np.uint64((1 << 64) - 1)
    IN = np.uint64(0)

    def halo(arr):
        payload = {p: arr[idx] for p, idx in send_idx.items()}
        allp = [None] * world
        dist.all_gather_object(allp, payload)
        for q in range(world):
            if q != rank and req[q]:
                arr[n_own + recv_off[q]:n_own + recv_off[q + 1]] = allp[q][rank]

    gid = np.arange(lo, hi, dtype=np.int64)
    T = np.full(nt, OUT, dtype=np.uint64)
    T[:n_own] = pins.np_words(0, gid, n, seed)
    M = np.full(nt, OUT, dtype=np.uint64)
    und = np.ones(n_own, dtype=bool)
    it = 0
    while True:
        tot = torch.tensor([int(und.sum())])
        dist.all_reduce(tot)
        if it > 0 and int(tot) == 0:
            break
        if it == 0 and int(tot) == 0:
            break
        halo(T)                                            # ghost T before Refresh Column
        m_own = np.minimum.reduceat(T[cols], starts) if n_own else np.zeros(0, np.uint64)
        M[:n_own] = np.where(m_own == IN, OUT, m_own)
        halo(M)                                            # ghost M before Decide
        any_out = np.maximum.reduceat((M[cols] == OUT).astype(np.int8), starts) > 0 if n_own else und
        all_eq = np.minimum.reduceat((M[cols] == T[rows]).astype(np.int8), starts) > 0 if n_own else und
        newT = T.copy()
        newT[:n_own][und & any_out] = OUT
        newT[:n_own][und & ~any_out & all_eq] = IN
        stay = und & ~any_out & ~all_eq
        newT[:n_own][stay] = pins.np_words(it + 1, gid[stay], n, seed)
        T = newT
        und = (T[:n_own] != IN) & (T[:n_own] != OUT)
        it += 1
    ins = [None] * world
    dist.all_gather_object(ins, (T[:n_own] == IN))
    if rank == 0:
        np.save(os.path.join(outdir, f"{name}_{seed}.npy"), np.concatenate([np.asarray(x, bool) for x in ins]))
        with open(os.path.join(outdir, f"{name}_{seed}.it"), "w") as fh:
            fh.write(str(it))
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1", "lap", "er", "kron", "elast"])
@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_protocol_gloo(name, world, tmp_path):
    import torch.multiprocessing as mp
    seed = 0 if world == 2 else 12345
    mp.spawn(_rank_main, args=(world, _free_port(), name, seed, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / f"{name}_{seed}.npy")
    its = int((tmp_path / f"{name}_{seed}.it").read_text())
    g = _graphs()[name]
    o = O.mis2(g.rowptr, g.colinds, seed=seed)
    assert np.array_equal(got, o.in_set) and its == o.iterations


def _agg_rank_main(rank, world, port, name, seed, outdir):
    """Alg. 3 over the partition with the exchange schedule of
    csrc/dist.cu dist_aggregate_run: global root numbering by an allgather of
    per-rank counts, halos of root ids / labels before the passes that read
    them, phase-3 aggregate sizes summed by an allreduce."""
    import torch.distributed as dist

    import paper_2204_02934_b200 as m
    import pins

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = _graphs()[name]
    n = g.n
    lo, hi = n * rank // world, n * (rank + 1) // world
    n_own = hi - lo
    ghosts, req, loc = m.plan_part(n, world, rank, g.rowptr[lo:hi + 1], g.colinds)
    recv_off = np.concatenate([[0], np.cumsum(req)])
    mine = [ghosts[recv_off[q]:recv_off[q + 1]] for q in range(world)]
    allreq = [None] * world
    dist.all_gather_object(allreq, mine)
    send_idx = {p: np.asarray(allreq[p][rank], dtype=np.int64) - lo for p in range(world) if p != rank}
    nt = n_own + len(ghosts)
    rp = g.rowptr[lo:hi + 1] - g.rowptr[lo]
    loc = loc.astype(np.int64)
    nbrs = [loc[rp[v]:rp[v + 1]] for v in range(n_own)]          # open rows (local ids)
    nbrs = [x[x != v] for v, x in enumerate(nbrs)]
    gid = np.arange(lo, hi, dtype=np.int64)
    OUT = np.uint64((1 << 64) - 1)
    IN = np.uint64(0)

    def halo(arr):
        payload = {p: arr[idx] for p, idx in send_idx.items()}
        allp = [None] * world
        dist.all_gather_object(allp, payload)
        for q in range(world):
            if q != rank and req[q]:
                arr[n_own + recv_off[q]:n_own + recv_off[q + 1]] = allp[q][rank]

    def global_offset(k):
        cnts = [None] * world
        dist.all_gather_object(cnts, int(k))
        return sum(cnts[:rank]), sum(cnts)

    def part_mis2(active_own):
        act = np.zeros(nt, dtype=bool)
        act[:n_own] = active_own
        halo(act)
        T = np.full(nt, OUT, dtype=np.uint64)
        T[:n_own][active_own] = pins.np_words(0, gid[active_own], n, seed)
        und = active_own.copy()
        it = 0
        while True:
            tot = torch.tensor([int(und.sum())])
            dist.all_reduce(tot)
            if int(tot) == 0:
                break
            halo(T)
            M = np.full(nt, OUT, dtype=np.uint64)
            for v in np.nonzero(active_own)[0]:
                cl = np.append(nbrs[v], v)
                cl = cl[act[cl]]
                mv = T[cl].min()
                M[v] = OUT if mv == IN else mv
            halo(M)
            newT = T.copy()
            for v in np.nonzero(und)[0]:
                cl = np.append(nbrs[v], v)
                cl = cl[act[cl]]
                if (M[cl] == OUT).any():
                    newT[v] = OUT
                elif (M[cl] == T[v]).all():
                    newT[v] = IN
                else:
                    newT[v] = pins.np_words(it + 1, gid[v:v + 1], n, seed)[0]
            T = newT
            und = active_own & (T[:n_own] != IN) & (T[:n_own] != OUT)
            it += 1
        return T[:n_own] == IN

    # phase 1
    in1 = part_mis2(np.ones(n_own, dtype=bool))
    off1, n1 = global_offset(in1.sum())
    R = np.full(nt, -1, dtype=np.int64)
    R[:n_own][in1] = off1 + np.arange(int(in1.sum()))
    halo(R)
    lab = np.full(nt, -1, dtype=np.int64)
    for v in range(n_own):
        if in1[v]:
            lab[v] = R[v]
        else:
            r = R[nbrs[v]]
            r = r[r >= 0]
            assert len(set(r.tolist())) <= 1
            if len(r):
                lab[v] = r[0]
    # phase 2
    in2 = part_mis2(lab[:n_own] < 0)
    halo(lab)
    acc = np.array([bool(in2[v]) and int((lab[nbrs[v]] < 0).sum()) >= 2 for v in range(n_own)], dtype=bool)
    off2, n2 = global_offset(acc.sum())
    A = np.full(nt, -1, dtype=np.int64)
    A[:n_own][acc] = n1 + off2 + np.arange(int(acc.sum()))
    halo(A)
    for v in range(n_own):
        if lab[v] >= 0:
            continue
        if acc[v]:
            lab[v] = A[v]
        else:
            a = A[nbrs[v]]
            a = a[a >= 0]
            if len(a):
                lab[v] = a[0]
    # phase 3
    halo(lab)
    tent = lab.copy()
    na = n1 + n2
    size = torch.from_numpy(np.bincount(tent[:n_own][tent[:n_own] >= 0], minlength=na).astype(np.int64))
    dist.all_reduce(size)
    size = size.numpy()
    for v in range(n_own):
        if tent[v] >= 0:
            continue
        cand = tent[nbrs[v]]
        cand = cand[cand >= 0]
        best = None
        for a in sorted(set(cand.tolist())):
            key = (-int((cand == a).sum()), int(size[a]), a)
            best = key if best is None or key < best else best
        lab[v] = best[2]
    labs = [None] * world
    dist.all_gather_object(labs, lab[:n_own])
    # coarse graph (csrc/dist.cu dist_coarsen_run): ghost labels, the coarse
    # edges of this rank's rows, allgather, union per coarse row
    halo(lab)
    edges = {(int(lab[v]), int(lab[w])) for v in range(n_own) for w in nbrs[v] if lab[v] != lab[w]}
    alle = [None] * world
    dist.all_gather_object(alle, sorted(edges))
    if rank == 0:
        merged = sorted(set().union(*[set(map(tuple, e)) for e in alle]))
        np.save(os.path.join(outdir, f"coarse_{name}_{seed}.npy"), np.asarray(merged, dtype=np.int64).reshape(-1, 2))
        np.save(os.path.join(outdir, f"agg_{name}_{seed}.npy"), np.concatenate(labs))
        with open(os.path.join(outdir, f"agg_{name}_{seed}.na"), "w") as fh:
            fh.write(str(na))
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["c1", "lap", "er", "elast"])
@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_aggregation_protocol_gloo(name, world, tmp_path):
    """Alg. 3 and the coarse graph under the partitioned exchange schedule ==
    monolithic oracle."""
    import torch.multiprocessing as mp
    seed = 0 if world == 2 else 777
    mp.spawn(_agg_rank_main, args=(world, _free_port(), name, seed, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / f"agg_{name}_{seed}.npy")
    na = int((tmp_path / f"agg_{name}_{seed}.na").read_text())
    g = _graphs()[name]
    o = O.aggregate(g.rowptr, g.colinds, seed=seed)
    assert na == o.num_aggs and np.array_equal(got, o.labels)
    crow, ccol = O.coarsen(g.rowptr, g.colinds, o.labels, o.num_aggs)
    want = np.stack([np.repeat(np.arange(o.num_aggs), np.diff(crow)), ccol], axis=1) if len(ccol) else np.zeros((0, 2))
    assert np.array_equal(np.load(tmp_path / f"coarse_{name}_{seed}.npy"), want)

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

/*
 * mis2.h -- C ABI of libmis2.so, the B200 (sm_100a) implementation of the
 * data-parallel hot path of Kelley & Rajamanickam, "Parallel, Portable
 * Algorithms for Distance-2 Maximal Independent Set and Graph Coarsening"
 * (arXiv 2204.02934).  "P:n" = PAPER.md line n.
 *
 * Conventions (all entry points)
 * ------------------------------
 *  - Graphs are CSR in DEVICE memory: rowptr int64[n+1] -- or int32[n+1]
 *    with rowptr_bits = 32 -- (rowptr[0] = 0, nondecreasing), colinds
 *    int32[nnz].  The graph must be symmetric, in
 *    range and duplicate free; a stored diagonal is allowed and ignored
 *    ("CRS"; reading Q23).  Row order inside a row is free
 *    except for mis2_validate_graph, which also requires sorted rows.
 *    0 <= n <= 2^31 - 3.
 *  - Every output array is a caller-owned device buffer; the library
 *    allocates nothing per call.  Scratch comes from the caller's workspace
 *    `ws` (device memory, >= mis2_workspace_size(...) bytes, 256-byte
 *    aligned).  Workspace contents need not be initialised.
 *  - All device work is enqueued on `stream` (a cudaStream_t; NULL = legacy
 *    default stream).  Functions returning host scalars synchronise that
 *    stream before returning; device outputs are then complete.  The *_async
 *    variants do not synchronise and write their scalars to device memory.
 *  - Calls with disjoint workspaces and outputs may run concurrently.
 *  - Return value: MIS2_OK (0) or a negative MIS2_E* code; no exception or
 *    abort crosses the ABI.  mis2_strerror() names a code,
 *    mis2_last_error() returns a thread-local detail string for the last
 *    failing call on the calling thread.
 */
#ifndef MIS2_H
#define MIS2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
#define MIS2_OK 0
#define MIS2_EINVAL (-1)         /* null pointer, n out of range, bad option      */
#define MIS2_ENOMEM (-2)         /* workspace smaller than mis2_workspace_size()   */
#define MIS2_ECUDA (-3)          /* CUDA runtime error (detail: mis2_last_error)   */
#define MIS2_ENCCL (-4)          /* NCCL error (distributed entry points)          */
#define MIS2_EGRAPH (-5)         /* VALIDATE failed: range / duplicate / asymmetry */
#define MIS2_ENOTCONVERGED (-6)  /* max_iters reached with undecided vertices      */
#define MIS2_ERANGE (-7)         /* output capacity too small; required size set   */
#define MIS2_EINTERNAL (-9)      /* an invariant of the algorithm failed           */

/* -------------------------------------------- priority schemes */
#define MIS2_SCHEME_XORSTAR 0 /* h(i,v) = f(f(i ^ seed) ^ f(v)), f = xorshift64*   */
#define MIS2_SCHEME_FIXED 1   /* Bell et al. fixed priorities: f(seed ^ f(v))     */
#define MIS2_SCHEME_XOR 2     /* as XORSTAR with f = plain xorshift64     */

/* -------------------------------------------------------------- op codes */
#define MIS2_OP_MIS2 0      /* mis2 / mis2_async                            */
#define MIS2_OP_AGGREGATE 1 /* mis2_aggregate                               */
#define MIS2_OP_COARSEN 2   /* mis2_coarsen                                 */
#define MIS2_OP_MIS2_HOST 3 /* mis2_host (graph staged through the workspace) */
#define MIS2_OP_VALIDATE 4  /* mis2_validate_graph                          */
#define MIS2_OP_COLOR 5     /* mis2_color                                   */

/* ------------------------------------------------------------------- flags */
#define MIS2_FLAG_VALIDATE 0x1u  /* run mis2_validate_graph first (EGRAPH on failure) */
#define MIS2_FLAG_BASIC 0x4u     /* mis2_aggregate: Alg. 2 "Basic MIS-2 Coarsening"
                                    instead of Alg. 3; leftovers join the aggregate of their
                                    smallest-id aggregated neighbour (reading Q28) */
#define MIS2_FLAG_PUSH_DECIDE 0x8u  /* force the push form of Decide (P:96-104 restated: the column
                                       pass marks N[w] of every w whose M_w becomes OUT and counts
                                       w for its argmin; Decide then reads no neighbour).  Default:
                                       push iff nnz/n >= 32.  Never changes results. */
#define MIS2_FLAG_PULL_DECIDE 0x10u /* force the pull form (Alg. 1 as written).  Never changes results. */
#define MIS2_FLAG_KEYS 0x20u     /* use 32-bit column keys (top 32 bits of the status word, ties
                                    resolved on the full words): half the gather bytes, for
                                    random-access graphs whose status words exceed L2.  Default:
                                    used iff 8n > 64 MB and the largest degree exceeds 16x the
                                    average.  Never changes results. */
#define MIS2_FLAG_NO_KEYS 0x40u  /* never use the 32-bit column keys.  Never changes results. */
#define MIS2_FLAG_WORD32 0x80u  /* status words of the paper's width W = 32 (Eq. 1;
                                    reading Q32): undecided T_v = (h32 & ~(2^b - 1)) | (v + 1) with
                                    h32 = the HIGH 32 bits of h, IN = 0, OUT = 2^32 - 1.  Requires
                                    b = ceil(log2(n + 2)) <= 31 (else MIS2_EINVAL).  Changes results
                                    (fewer priority bits, more ties broken by id); stored
                                    zero-extended in the 64-bit arrays, which orders every word
                                    exactly as 32-bit storage would (results identical to a
                                    32-bit implementation).  MIS-2 / aggregation / partitioned. */
#define MIS2_FLAG_ITER_STATS 0x100u /* mis2_aggregate: `stats` holds 8 + 12 * max_iters int64: after the
                                       8 summary entries, the per-iteration worklist statistics (as
                                       mis2()'s `stats`, max_iters rows of 6) of the phase-1 MIS-2, then of
                                       the masked phase-2 MIS-2 (instrumented, slower runs; measurement) */
#define MIS2_FLAG_TIMELINE 0x2u  /* measurement aid: mis2()'s `stats` receives int64 device
                                    timestamps (ns, %globaltimer) taken by block 0 after
                                    the init phase and after every grid barrier:
                                    [init, col0, dec0, col1, dec1, ...]; stats must hold
                                    2 * max_iters + 2 entries */

typedef struct {
    int64_t n;              /* |V|                                         */
    int64_t nnz;            /* stored entries = rowptr[n]                  */
    union {
        const int64_t* rowptr;    /* device int64[n+1] (rowptr_bits 0 or 64) */
        const int32_t* rowptr32;  /* device int32[n+1] (rowptr_bits 32)      */
    };
    const int32_t* colinds; /* device int32[nnz]                           */
    int32_t rowptr_bits;    /* 0 or 64: int64 row pointers; 32: int32 row pointers
                               (nnz < 2^31), widened into the workspace on entry by
                               mis2 / mis2_async / mis2_aggregate / mis2_coarsen /
                               mis2_validate_graph (the workspace sizes include it);
                               other entry points: MIS2_EINVAL.  Anything else:
                               MIS2_EINVAL. */
    int32_t reserved;       /* 0 */
} mis2_graph;

typedef struct {
    uint64_t seed;      /* hash seed, mixed as f(iter ^ seed) (reading Q4); default 0 */
    int32_t max_iters;  /* <= 0: 10*b + 20 with b = ceil(log2(n+2)) (reading Q12)     */
    int32_t scheme;     /* MIS2_SCHEME_*                                              */
    uint32_t flags;     /* MIS2_FLAG_*                                                */
    int32_t group;      /* lanes per CSR row in the neighbour loops: 0 = auto, else
                           1,2,4,8,16,32 (§V-D "SIMD"); never changes results */
    /* TEST ONLY (Fig. 1 replay): when non-NULL, iteration i <
       prio_iters uses T_v = (prio_override[i*n + v] << b) | (v + 1) instead
       of the hash.  Device memory, uint64[prio_iters * n]. */
    const uint64_t* prio_override;
    int32_t prio_iters;
    int32_t reserved;
} mis2_opts;

/* Fill *o with the defaults (seed 0, Xor*, auto everything). */
void mis2_opts_default(mis2_opts* o);

/* Workspace bytes needed for `op` (MIS2_OP_*) on a graph of n vertices and
 * nnz stored entries on the CURRENT device.  MIS2_OK or MIS2_EINVAL. */
int mis2_workspace_size(int64_t n, int64_t nnz, int32_t op, size_t* bytes);

/*
 * MIS-2 -- Alg. 1 "MIS-2: Kokkos Kernels Algorithm" (§III-A) with
 * the §V optimisations: per-iteration xorshift* priorities, the two
 * worklists, 64-bit compressed status words IN = 0 < (priority
 * << b | id+1) < OUT = 2^64-1 (Eq. 1), closed neighbourhoods
 * (reading Q1) and decide on the pre-update T_v (reading Q2).
 *
 *   in_set : device uint8[n]; 1 iff v is in the MIS-2 ({v : T_v = IN})
 *   count  : host; |MIS-2|
 *   iters  : host; loop bodies executed ("number of times the loop
 *            ... is executed")
 *   stats  : host int64[max_iters * 6] or NULL.  When non-NULL the call
 *            also records, per iteration, |worklist1|, |worklist2|, E1, E2
 *            (sums of stored row lengths over the lists) and |N[wl1]|,
 *            |N[wl2]| (distinct closed-neighbourhood vertices) -- a slower
 *            instrumented run used for the algorithmic-byte model.
 * Returns MIS2_ENOTCONVERGED with in_set = vertices IN so far and
 * *iters = max_iters when worklist1 is not empty after max_iters loops.
 */
int mis2(const mis2_graph* g, const mis2_opts* o, uint8_t* in_set, int64_t* count, int32_t* iters,
         int64_t* stats, void* ws, size_t ws_bytes, void* stream);

/* Same as mis2() without synchronisation: *d_count (int64), *d_iters
 * (int32) and *d_status (int32, MIS2_OK / MIS2_ENOTCONVERGED) are DEVICE
 * pointers written by the last kernel.  Argument errors are still returned. */
int mis2_async(const mis2_graph* g, const mis2_opts* o, uint8_t* in_set, int64_t* d_count,
               int32_t* d_iters, int32_t* d_status, void* ws, size_t ws_bytes, void* stream);

/* End-to-end variant with HOST buffers: rowptr_h int64[n+1] and colinds_h
 * int32[nnz] (pinned for full speed) are copied into the workspace, MIS-2
 * runs, and in_set_h uint8[n] is copied back.  ws from MIS2_OP_MIS2_HOST. */
int mis2_host(int64_t n, int64_t nnz, const int64_t* rowptr_h, const int32_t* colinds_h,
              const mis2_opts* o, uint8_t* in_set_h, int64_t* count, int32_t* iters, void* ws,
              size_t ws_bytes, void* stream);

/*
 * MIS-2 aggregation -- Alg. 3 (§III-B):
 *   phase 1: roots = MIS2(G); each root and its neighbours form an aggregate,
 *            numbered by ascending root id (reading Q18);
 *   phase 2: MIS2 of the subgraph induced by unaggregated vertices (same
 *            seed, original ids, iter from 0 -- reading Q15); a root with
 *            >= 2 unaggregated neighbours aggregates them (Q16-Q17);
 *   phase 3: frozen tentative labels; every leftover joins the adjacent
 *            aggregate of max coupling, then min size, then min id
 *            (reading Q19).
 *   labels   : device int32[n], aggregate of each vertex, in [0, num_aggs)
 *   num_aggs : host
 *   roots    : device int32[n] or NULL; roots[a] = root vertex of aggregate a
 *   stats    : host int64[8] or NULL: |M1|, iters1, |M2|, iters2, accepted
 *              phase-2 roots, phase-3 leftovers, n1, num_aggs
 * Repeated calls with the same graph pointers, sizes, outputs, workspace and
 * options (graphs with 8n <= 64 MB and no per-iteration statistics) replay
 * the call's launch sequence as one CUDA graph captured on the second such
 * call; it runs on a library-owned stream per device, ordered after and
 * before the caller's stream by events (calls from several threads then
 * serialise on that stream).  MIS2_AGG_GRAPH=0 in the environment disables it.
 */
int mis2_aggregate(const mis2_graph* g, const mis2_opts* o, int32_t* labels, int64_t* num_aggs,
                   int32_t* roots, int64_t* stats, void* ws, size_t ws_bytes, void* stream);

/*
 * Coarse graph A_c <- coarsen(A) (Alg. 4 setup): vertices are the
 * aggregates; (a,b), a != b, is an entry iff some stored fine entry (u,v)
 * has labels[u] = a, labels[v] = b.  Rows sorted, deduplicated, no
 * self-loops (reading Q21).
 *   labels    : device int32[n], values in [0, num_aggs)
 *   c_rowptr  : device int64[num_aggs + 1] -- always written
 *   c_colinds : device int32[cap] -- written only when cap >= nnz_c
 *   c_nnz     : host; stored coarse entries.  MIS2_ERANGE when cap < nnz_c
 *               (two-call convention: query with cap = 0, allocate, repeat).
 */
int mis2_coarsen(const mis2_graph* g, const int32_t* labels, int64_t num_aggs, int64_t* c_rowptr,
                 int32_t* c_colinds, int64_t cap, int64_t* c_nnz, void* ws, size_t ws_bytes,
                 void* stream);

/* Check the input contract on the device: rowptr monotone with rowptr[n] =
 * nnz, colinds in range, rows sorted without duplicates, pattern symmetric.
 * MIS2_OK or MIS2_EGRAPH (detail in mis2_last_error()). */
int mis2_validate_graph(const mis2_graph* g, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Partitioned MIS-2 (1-D row partition).  Part q of P owns
 * rows [n*q/P, n*(q+1)/P).  Before every Refresh Column the ghost T values
 * are exchanged, before every Decide the ghost M values, after every Decide
 * |worklist_1| is summed over the parts; hashes use global ids and b
 * uses the global n, so the result is bit-identical to mis2() on one GPU
 * (each phase reads only the previous phase's arrays).
 *
 * A mis2_comm owns its communicator and the device copies of its parts
 * (allocated by mis2_comm_set_graph, freed by mis2_comm_destroy).
 *   NCCL : one process per GPU; rank 0 gets the id from mis2_comm_unique_id,
 *          broadcasts it (e.g. torch.distributed), every rank calls
 *          mis2_comm_init_nccl on its current device.  set_graph takes this
 *          rank's rows: rowptr_h[n_own + 1], colinds_h[rowptr_h[0] ..
 *          rowptr_h[n_own]) with GLOBAL column ids (collective call).
 *          mis2_dist_mis2's in_set is the rank's n_own-entry device mask.
 *   LOCAL: all P parts in this process on the current device (halos copied
 *          device to device): set_graph takes the whole host CSR; in_set is
 *          the global n-entry mask.  Same algorithm, for testing and for
 *          graphs partitioned on one GPU.
 * ---------------------------------------------------------------------- */
typedef struct mis2_comm mis2_comm;
int mis2_comm_unique_id(uint8_t* id128);
int mis2_comm_init_nccl(const uint8_t* id128, int nranks, int rank, mis2_comm** out);
int mis2_comm_init_local(int nparts, mis2_comm** out);
int mis2_comm_set_graph(mis2_comm* c, int64_t n_global, const int64_t* rowptr_h, const int32_t* colinds_h,
                        void* stream);
/* One launch of the partitioned persistent kernel per call (halo words
 * stored straight into the peers' ghost slots, partitions meeting at a
 * device-side mailbox barrier).  If a peer partition does not post at a
 * barrier within 10 s (a GPU of the job gone or hung) the call gives up and
 * returns MIS2_EINTERNAL instead of hanging; the communicator is then
 * unusable. */
int mis2_dist_mis2(mis2_comm* c, const mis2_opts* o, uint8_t* in_set, int64_t* count, int32_t* iters,
                   void* stream);
/* Alg. 3 over the partition, bit-identical to mis2_aggregate():
 * both MIS-2 calls partitioned, roots numbered by a global exclusive prefix
 * of per-part counts (allgather), root / accepted-root ids and labels
 * exchanged as ghost halos before the passes that read them, phase-3
 * aggregate sizes summed over the parts (allreduce).  labels: device int32,
 * this rank's n_own rows (NCCL) or all n rows (LOCAL), GLOBAL aggregate ids.
 * stats (host int64[8] or NULL) as mis2_aggregate's.  Collective call.
 * MIS2_FLAG_BASIC and prio_override are not supported (MIS2_EINVAL). */
int mis2_dist_aggregate(mis2_comm* c, const mis2_opts* o, int32_t* labels, int64_t* num_aggs, int64_t* stats,
                        void* stream);
/* Coarse graph of the partitioned graph given its aggregate labels
 * (as produced by mis2_dist_aggregate: this rank's rows (NCCL) or all rows
 * (LOCAL), global ids in [0, num_aggs)).  Every part builds the coarse edges
 * of its own rows (ghost labels exchanged first); the per-part coarse CSRs
 * are allgathered and merged, so the result -- identical to mis2_coarsen()
 * on the whole graph -- is REPLICATED on every rank: c_rowptr int64
 * [num_aggs + 1] and c_colinds int32 [cap], device.  Two-call convention as
 * mis2_coarsen (MIS2_ERANGE with *c_nnz set when cap is too small; c_colinds
 * may be NULL).  Scratch comes from the communicator's pool: allocated when
 * a call first needs it (or more of it), kept for later calls, freed with
 * the graph (mis2_comm_set_graph / mis2_comm_destroy).  Collective call. */
int mis2_dist_coarsen(mis2_comm* c, const int32_t* labels, int64_t num_aggs, int64_t* c_rowptr,
                      int32_t* c_colinds, int64_t cap, int64_t* c_nnz, void* stream);
/* rows [lo, hi) and ghost count of local part `part` (NCCL: part 0) */
int mis2_comm_part_info(mis2_comm* c, int part, int64_t* lo, int64_t* hi, int64_t* n_ghost);
int mis2_comm_destroy(mis2_comm* c);

/* Host-only partition planner (no device, no communicator): part `part` of
 * `nparts` with rows rowptr_local[n_own+1] and GLOBAL column ids.  Returns the
 * number of ghosts, their sorted global ids (ghost_ids may be NULL), the
 * number requested from each owner (req_counts[nparts]) and the columns in
 * the local index space [owned | ghosts] (colinds_local may be NULL). */
int mis2_plan_part(int64_t n_global, int nparts, int part, const int64_t* rowptr_local,
                   const int32_t* colinds_global, int64_t* n_ghost, int64_t* ghost_ids, int64_t* req_counts,
                   int32_t* colinds_local);

/* ------------------------------------------------------------------------
 * Alg. 4 "Cluster Multicolor Gauss-Seidel" (§III-C).
 *
 * mis2_color: deterministic greedy colouring of a graph (reading Q30:
 * Jones-Plassmann rounds, priorities = the MIS-2 status words of iteration 0
 * with `seed`; every vertex takes the smallest colour none of its
 * earlier-coloured neighbours has).  color: device int32[n]; *ncolors on
 * return (synchronises the stream).  Scratch from the caller's workspace
 * ws (>= mis2_workspace_size(n, nnz, MIS2_OP_COLOR) bytes).
 *
 * mis2_cgs_setup: Alg. 4's setup.  labels (device int32[n]) and
 * num_aggs give the clusters (e.g. mis2_aggregate), `coarse` their coarse
 * graph (mis2_coarsen; device CSR with num_aggs rows), coloured with
 * mis2_color; labels == NULL gives point multicolor Gauss-Seidel (every row
 * its own cluster, the graph itself coloured).  vals: device f64[nnz], A_ii
 * must be stored and nonzero (MIS2_EINVAL otherwise).  g, vals must stay
 * valid while the handle is used; the handle owns its cluster / colour-set
 * arrays and the setup scratch -- one device allocation made by the setup
 * call, freed by mis2_cgs_destroy (the apply calls allocate nothing).
 *
 * mis2_cgs_apply: `sweeps` sweeps on x (device f64[n], in place) for the
 * right-hand side b (device f64[n]): direction 1 forward (colours and rows
 * ascending), 2 backward (both descending), 0 symmetric (forward then
 * backward).  Row update x_i += (b_i - A_i x) / A_ii (reading Q31).  Clusters
 * of one colour are updated concurrently; enqueued on `stream`.
 * ---------------------------------------------------------------------- */
typedef struct mis2_cgs mis2_cgs;
int mis2_color(const mis2_graph* g, uint64_t seed, int32_t* color, int32_t* ncolors, void* ws, size_t ws_bytes,
               void* stream);
int mis2_cgs_setup(const mis2_graph* g, const double* vals, const int32_t* labels, int64_t num_aggs,
                   const mis2_graph* coarse, uint64_t seed, mis2_cgs** out, void* stream);
int mis2_cgs_ncolors(const mis2_cgs* h);
int mis2_cgs_apply(mis2_cgs* h, const double* b, double* x, int sweeps, int direction, void* stream);
int mis2_cgs_destroy(mis2_cgs* h);

/* Number of kernel launches issued by the last call on this thread
 * (measurement aid for bench.py's "gpu_launches"). */
int64_t mis2_last_launch_count(void);

const char* mis2_strerror(int status);
const char* mis2_last_error(void);
/* Library build string (arch, git-independent version). */
const char* mis2_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MIS2_H */

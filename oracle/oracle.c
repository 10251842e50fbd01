/*
 * oracle/oracle.c -- plain, slow, serial CPU oracle for the MIS-2 hot path of
 * Kelley & Rajamanickam, "Parallel, Portable Algorithms for Distance-2 Maximal
 * Independent Set and Graph Coarsening" (arXiv 2204.02934).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_2204_02934_b200/), and neither imports the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / algorithm in
 * brackets); "Qk" = the reading of an ambiguous passage listed in DESIGN.md
 * (the same numbering as SURVEY.md §8(c).2).
 *
 * Everything is written in the paper's order and notation: worklists are
 * ascending vertex lists, every phase is a plain loop, no blocking or fusion.
 * Pins (tests/test_oracle_*.py): Fig. 1 replay (P1), brute-force distance-2
 * independence + maximality (P2), Luby-on-G^2 (P3), worklist-free Bell-style
 * sweep (P4), closed forms (P5), hash vectors (P6), packing (P7),
 * tab:structured-scaling quality (P8), aggregation invariants (P10),
 * pattern(P^T A P) via scipy (P11), diagonal invariance (P12).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL -1
#define ORC_ENOMEM -2
#define ORC_ENOTCONVERGED -6
#define ORC_EASSERT -9

/* Priority schemes of tab:rng-iterations. */
#define ORC_SCHEME_XORSTAR 0 /* h(i,v) = f(f(i^seed) ^ f(v)), f = xorshift64*  (used) */
#define ORC_SCHEME_FIXED 1   /* Bell et al.: priorities drawn once: f(seed ^ f(v)) */
#define ORC_SCHEME_XOR 2     /* same as XORSTAR with f = plain xorshift64 */
/* Scheme modifier: status words of the paper's width W = 32 ("the
 * same width as the vertex ids"; reading Q32): the priority is taken from the
 * high 32 bits of h, IN = 0, OUT = 2^32 - 1.  Needs b <= 31. */
#define ORC_WORD32 0x10

/* ---------------------------------------------------------------------------
 * §V-A Pseudo-random priorities: "h(iter, v) = f(f(iter) ⊕ f(v))";
 * "for Xor*, f(x) is the 64-bit xorshift* (xorshift followed by a linear
 * congruential step)".  Constants: reading Q3 (Marsaglia's (13,7,17) triple,
 * multiplier 0x2545F4914F6CDD1D); seed mixing: reading Q4.
 * ------------------------------------------------------------------------- */
uint64_t orc_xorshift64(uint64_t x) {
    x ^= x << 13;
    x ^= x >> 7;
    x ^= x << 17;
    return x;
}

uint64_t orc_xorshift64star(uint64_t x) { return orc_xorshift64(x) * 0x2545F4914F6CDD1DULL; }

uint64_t orc_h(int scheme, uint64_t iter, uint64_t v, uint64_t seed) {
    if (scheme == ORC_SCHEME_FIXED) return orc_xorshift64star(seed ^ orc_xorshift64star(v));
    if (scheme == ORC_SCHEME_XOR) return orc_xorshift64(orc_xorshift64(iter ^ seed) ^ orc_xorshift64(v));
    return orc_xorshift64star(orc_xorshift64star(iter ^ seed) ^ orc_xorshift64star(v));
}

/* ---------------------------------------------------------------------------
 * §V-C Compressed status tuples (Eq. 1): IN = 0, OUT = UINT_MAX,
 * undecided = (priority << b) | (id + 1), b = ceil(log2(|V| + 2)).
 * Word width 64 (reading Q6); b = bitlength(n + 1) (reading Q7); the priority
 * field is the HIGH 64-b bits of h (reading Q5).
 * ------------------------------------------------------------------------- */
#define ORC_IN 0ULL
#define ORC_OUT 0xFFFFFFFFFFFFFFFFULL

int orc_bits(int64_t n) {
    /* smallest b with 2^b >= n + 2  ( = ceil(log2(n+2)) ) */
    int b = 0;
    while (b < 63 && ((int64_t)1 << b) < n + 2) b++;
    return b;
}

uint64_t orc_pack(uint64_t priority, int64_t id, int b) { return (priority << b) | (uint64_t)(id + 1); }

uint64_t orc_word(int scheme, uint64_t iter, int64_t v, uint64_t seed, int b) {
    uint64_t h = orc_h(scheme & ~ORC_WORD32, iter, (uint64_t)v, seed);
    if (scheme & ORC_WORD32) h >>= 32; /* a W = 32 hash: the high half of h (Q5, Q32) */
    return orc_pack(h >> b, v, b);     /* = (h & ~(2^b - 1)) | (v + 1) */
}

/* ---------------------------------------------------------------------------
 * Alg. 1 "MIS-2: Kokkos Kernels Algorithm" (§III-A).
 *
 * adj(v) is the CLOSED neighbourhood N[v] (reading Q1, from Fig. 1 P:151 and
 * Lemma 1's self-loops P:361); stored diagonal entries are harmless repeats.
 * Decide evaluates both conditions on the pre-update T_v (reading Q2).
 * active == NULL: every vertex takes part.  Otherwise only active vertices
 * take part and inactive ones are invisible (induced subgraph, phase 2 of
 * Alg. 3, reading Q15).
 *
 * prio_override (test only): iteration i < prio_iters uses the priority
 * prio_override[i*n + v] in place of h, i.e. T_v = (p << b) | (v+1)
 * (Fig. 1 replay).
 *
 * stats (optional, int64[max_iters * 6]): per iteration |wl1|, |wl2|,
 * E1 = sum of stored row lengths over wl1, E2 (same over wl2),
 * |N[wl1]| and |N[wl2]| (distinct closed-neighbourhood vertices).
 * T_out / M_out (optional, uint64[n]): final status arrays.
 *
 * Returns ORC_OK, or ORC_ENOTCONVERGED (in_set = vertices IN so far,
 * *iters = max_iters) when the loop has not emptied worklist_1.
 * ------------------------------------------------------------------------- */
int orc_mis2(int64_t n, const int64_t* rowptr, const int32_t* colinds, uint64_t seed, int scheme,
             int32_t max_iters, const uint8_t* active, const uint64_t* prio_override, int32_t prio_iters,
             uint8_t* in_set, int64_t* count, int32_t* iters, int64_t* stats, uint64_t* T_out,
             uint64_t* M_out) {
    if (n < 0 || (n > 0 && (!rowptr || !colinds)) || !in_set || !count || !iters) return ORC_EINVAL;
    const int b = orc_bits(n);
    const uint64_t OUT = (scheme & ORC_WORD32) ? 0xFFFFFFFFULL : ORC_OUT; /* UINT_MAX of width W */
    if ((scheme & ORC_WORD32) && b > 31) return ORC_EINVAL;
    if (max_iters <= 0) max_iters = 10 * b + 20; /* reading Q12 */

    uint64_t* T = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n + 1));
    uint64_t* M = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n + 1));
    int64_t* wl1 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t* wl2 = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t* mark = stats ? (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1)) : NULL;
    if (!T || !M || !wl1 || !wl2 || (stats && !mark)) {
        free(T); free(M); free(wl1); free(wl2); free(mark);
        return ORC_ENOMEM;
    }
    if (mark) for (int64_t v = 0; v < n; v++) mark[v] = -1;

#define ACTIVE(w) (active == NULL || active[w])
    /* IN <- 0; OUT <- UINT_MAX.  Vertices outside worklist_2 keep
     * M = OUT (reading Q9); inactive vertices are never read. */
    for (int64_t v = 0; v < n; v++) { T[v] = OUT; M[v] = OUT; }
    /* worklist_1 <- 0..|V|, worklist_2 <- 0..|V| */
    int64_t n1 = 0, n2 = 0;
    for (int64_t v = 0; v < n; v++)
        if (ACTIVE(v)) { wl1[n1++] = v; wl2[n2++] = v; }
    int64_t iter = 0;
    int rc = ORC_OK;

    while (n1 > 0) {
        if (iter >= max_iters) { rc = ORC_ENOTCONVERGED; break; }
        if (stats) {
            int64_t e1 = 0, e2 = 0, d1 = 0, d2 = 0;
            for (int64_t k = 0; k < n1; k++) {
                int64_t v = wl1[k];
                e1 += rowptr[v + 1] - rowptr[v];
                if (mark[v] != 2 * iter) { mark[v] = 2 * iter; d1++; }
                for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++)
                    if (mark[colinds[j]] != 2 * iter) { mark[colinds[j]] = 2 * iter; d1++; }
            }
            for (int64_t k = 0; k < n2; k++) {
                int64_t v = wl2[k];
                e2 += rowptr[v + 1] - rowptr[v];
                if (mark[v] != 2 * iter + 1) { mark[v] = 2 * iter + 1; d2++; }
                for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++)
                    if (mark[colinds[j]] != 2 * iter + 1) { mark[colinds[j]] = 2 * iter + 1; d2++; }
            }
            int64_t* s = stats + 6 * iter;
            s[0] = n1; s[1] = n2; s[2] = e1; s[3] = e2; s[4] = d1; s[5] = d2;
        }

        /* Refresh row status: T_v <- h(iter, v) | v+1 */
        for (int64_t k = 0; k < n1; k++) {
            int64_t v = wl1[k];
            if (prio_override && iter < prio_iters)
                T[v] = orc_pack(prio_override[iter * n + v], v, b);
            else
                T[v] = orc_word(scheme, (uint64_t)iter, v, seed, b);
        }

        /* Refresh column status: M_v <- min(T_w : w in adj(v));
         * if M_v = IN then M_v <- OUT */
        for (int64_t k = 0; k < n2; k++) {
            int64_t v = wl2[k];
            uint64_t m = T[v]; /* closed neighbourhood: v itself (Q1) */
            for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++) {
                int64_t w = colinds[j];
                if (ACTIVE(w) && T[w] < m) m = T[w];
            }
            if (m == ORC_IN) m = OUT;
            M[v] = m;
        }

        /* Decide IN/OUT of set, on the pre-update T_v (Q2):
         * if exists w in adj(v): M_w = OUT  -> T_v <- OUT
         * else if forall w in adj(v): T_v = M_w -> T_v <- IN */
        for (int64_t k = 0; k < n1; k++) {
            int64_t v = wl1[k];
            const uint64_t tv = T[v];
            int any_out = (M[v] == OUT);
            int all_eq = (M[v] == tv);
            for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++) {
                int64_t w = colinds[j];
                if (!ACTIVE(w)) continue;
                if (M[w] == OUT) any_out = 1;
                if (M[w] != tv) all_eq = 0;
            }
            if (any_out) T[v] = OUT;
            else if (all_eq) T[v] = ORC_IN;
        }

        /* Compact worklists: ascending order kept */
        int64_t k1 = 0, k2 = 0;
        for (int64_t k = 0; k < n1; k++)
            if (T[wl1[k]] != ORC_IN && T[wl1[k]] != OUT) wl1[k1++] = wl1[k];
        for (int64_t k = 0; k < n2; k++)
            if (M[wl2[k]] != OUT) wl2[k2++] = wl2[k];
        n1 = k1;
        n2 = k2;
        iter++;
    }
#undef ACTIVE

    /* return {v : T_v = IN} */
    int64_t c = 0;
    for (int64_t v = 0; v < n; v++) {
        in_set[v] = (T[v] == ORC_IN);
        c += in_set[v];
    }
    *count = c;
    *iters = (int32_t)iter;
    if (T_out) memcpy(T_out, T, sizeof(uint64_t) * (size_t)n);
    if (M_out) memcpy(M_out, M, sizeof(uint64_t) * (size_t)n);
    free(T); free(M); free(wl1); free(wl2); free(mark);
    return rc;
}

/* ---------------------------------------------------------------------------
 * Alg. 3 "MIS-2 based Aggregation" (§III-B).
 *
 * labels int32[n] (UNAGG = -1 never remains on success); roots int32[n]
 * (optional): roots[a] = root vertex of aggregate a.
 * stats (optional, int64[8]): |M1|, iterations of M1, |M2|, iterations of
 * M2, accepted phase-2 roots, phase-3 leftovers, n1 (= |M1|), num_aggs.
 *
 * Readings: Q15 (phase-2 MIS-2 = masked Alg. 1 on original ids, same b and
 * seed, iter from 0), Q16 (">= 2 unagg. neighbors" counts distinct w != v
 * unaggregated after phase 1), Q17 (all unaggregated neighbours join),
 * Q18 (aggregate numbering ascending by root vertex, phase 1 first),
 * Q19 (phase-3 tie: max coupling, then min aggsize, then min id),
 * Q20 (every leftover has a candidate).
 * ------------------------------------------------------------------------- */
#define ORC_UNAGG (-1)

int orc_aggregate(int64_t n, const int64_t* rowptr, const int32_t* colinds, uint64_t seed, int scheme,
                  int32_t max_iters, int32_t* labels, int64_t* num_aggs, int32_t* roots, int64_t* stats) {
    if (n < 0 || !labels || !num_aggs) return ORC_EINVAL;
    int rc = ORC_OK;
    uint8_t* S = (uint8_t*)calloc((size_t)n + 1, 1);
    uint8_t* U = (uint8_t*)calloc((size_t)n + 1, 1);
    int32_t* tent = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    int32_t* rid = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    if (!S || !U || !tent || !rid) { rc = ORC_ENOMEM; goto done; }

    /* Phase 1: M1 <- MIS2(G); aggregate from v and its neighbours */
    int64_t c1 = 0;
    int32_t it1 = 0;
    rc = orc_mis2(n, rowptr, colinds, seed, scheme, max_iters, NULL, NULL, 0, S, &c1, &it1, NULL, NULL, NULL);
    if (rc != ORC_OK) goto done;
    int32_t na = 0;
    for (int64_t v = 0; v < n; v++) labels[v] = ORC_UNAGG;
    for (int64_t v = 0; v < n; v++) /* root ids: ascending vertex order (Q18) */
        if (S[v]) { rid[v] = na; if (roots) roots[na] = (int32_t)v; na++; }
    for (int64_t v = 0; v < n; v++) {
        if (S[v]) { labels[v] = rid[v]; continue; }
        for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++) {
            int64_t w = colinds[j];
            if (w != v && S[w]) {
                /* at most one root neighbour: roots are >= 3 apart */
                if (labels[v] != ORC_UNAGG && labels[v] != rid[w]) { rc = ORC_EASSERT; goto done; }
                labels[v] = rid[w];
            }
        }
    }
    const int32_t n1 = na;

    /* Phase 2: M2 <- MIS2(G \ {aggregated}) */
    for (int64_t v = 0; v < n; v++) U[v] = (labels[v] == ORC_UNAGG);
    int64_t c2 = 0;
    int32_t it2 = 0;
    memset(S, 0, (size_t)n);
    rc = orc_mis2(n, rowptr, colinds, seed, scheme, max_iters, U, NULL, 0, S, &c2, &it2, NULL, NULL, NULL);
    if (rc != ORC_OK) goto done;
    /* roots with >= 2 unaggregated neighbours are accepted, ascending (Q16, Q18) */
    int64_t accepted = 0;
    for (int64_t r = 0; r < n; r++) {
        if (!S[r]) continue;
        int64_t cnt = 0;
        for (int64_t j = rowptr[r]; j < rowptr[r + 1]; j++) {
            int64_t w = colinds[j];
            if (w != r && U[w]) cnt++;
        }
        if (cnt >= 2) {
            if (roots) roots[na] = (int32_t)r;
            labels[r] = na;
            for (int64_t j = rowptr[r]; j < rowptr[r + 1]; j++) {
                int64_t w = colinds[j];
                if (w != r && U[w]) {
                    /* conflicts impossible: M2 is distance-2 independent in G' (Q17) */
                    if (labels[w] != ORC_UNAGG) { rc = ORC_EASSERT; goto done; }
                    labels[w] = na;
                }
            }
            na++;
            accepted++;
        }
    }

    /* Phase 3: tent <- labels; coupling/aggsize from tent;
     * join max coupling, tie -> min aggsize (-> min id, Q19) */
    memcpy(tent, labels, sizeof(int32_t) * (size_t)n);
    int64_t* aggsize = (int64_t*)calloc((size_t)na + 1, sizeof(int64_t));
    int64_t* coupling = (int64_t*)calloc((size_t)na + 1, sizeof(int64_t));
    if (!aggsize || !coupling) { free(aggsize); free(coupling); rc = ORC_ENOMEM; goto done; }
    for (int64_t v = 0; v < n; v++)
        if (tent[v] != ORC_UNAGG) aggsize[tent[v]]++;
    int64_t leftovers = 0;
    for (int64_t v = 0; v < n; v++) {
        if (tent[v] != ORC_UNAGG) continue;
        leftovers++;
        /* coupling(a, v) = |{u : (u,v) in E and tent_u = a}| */
        for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++) {
            int64_t u = colinds[j];
            if (u != v && tent[u] != ORC_UNAGG) coupling[tent[u]]++;
        }
        int32_t best = ORC_UNAGG;
        for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++) {
            int64_t u = colinds[j];
            if (u == v || tent[u] == ORC_UNAGG) continue;
            int32_t a = tent[u];
            if (best == ORC_UNAGG || coupling[a] > coupling[best] ||
                (coupling[a] == coupling[best] &&
                 (aggsize[a] < aggsize[best] || (aggsize[a] == aggsize[best] && a < best))))
                best = a;
        }
        for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++) { /* reset the counters */
            int64_t u = colinds[j];
            if (u != v && tent[u] != ORC_UNAGG) coupling[tent[u]] = 0;
        }
        if (best == ORC_UNAGG) { rc = ORC_EASSERT; break; } /* Q20 */
        labels[v] = best;
    }
    free(aggsize);
    free(coupling);
    if (rc != ORC_OK) goto done;

    *num_aggs = na;
    if (stats) {
        stats[0] = c1; stats[1] = it1; stats[2] = c2; stats[3] = it2;
        stats[4] = accepted; stats[5] = leftovers; stats[6] = n1; stats[7] = na;
    }
done:
    free(S); free(U); free(tent); free(rid);
    return rc;
}

/* ---------------------------------------------------------------------------
 * Alg. 2 "Basic MIS-2 Coarsening" -- SURVEY §8(f) NEXT-1.
 * Roots = MIS-2 (ascending ids); each root and its neighbours form an
 * aggregate; every other vertex joins "any" adjacent aggregate -- made
 * deterministic as: the aggregate of its smallest-id phase-1-labelled
 * neighbour (reading Q28).
 * ------------------------------------------------------------------------- */
int orc_coarsen_basic(int64_t n, const int64_t* rowptr, const int32_t* colinds, uint64_t seed,
                      int scheme, int32_t max_iters, int32_t* labels, int64_t* num_aggs) {
    if (n < 0 || !labels || !num_aggs) return ORC_EINVAL;
    uint8_t* S = (uint8_t*)calloc((size_t)n + 1, 1);
    int32_t* tent = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    if (!S || !tent) { free(S); free(tent); return ORC_ENOMEM; }
    int64_t c = 0;
    int32_t it = 0;
    int rc = orc_mis2(n, rowptr, colinds, seed, scheme, max_iters, NULL, NULL, 0, S, &c, &it, NULL, NULL, NULL);
    int32_t na = 0;
    if (rc == ORC_OK) {
        for (int64_t v = 0; v < n; v++) labels[v] = ORC_UNAGG;
        for (int64_t v = 0; v < n; v++) if (S[v]) labels[v] = na++;
        for (int64_t v = 0; v < n; v++) {
            if (S[v]) continue;
            for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++) {
                int64_t w = colinds[j];
                if (w != v && S[w]) labels[v] = labels[w];
            }
        }
        memcpy(tent, labels, sizeof(int32_t) * (size_t)n);
        for (int64_t v = 0; v < n && rc == ORC_OK; v++) {
            if (tent[v] != ORC_UNAGG) continue;
            int64_t best_u = -1;
            for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++) {
                int64_t u = colinds[j];
                if (u != v && tent[u] != ORC_UNAGG && (best_u < 0 || u < best_u)) best_u = u;
            }
            if (best_u < 0) rc = ORC_EASSERT; /* maximality of MIS-2 */
            else labels[v] = tent[best_u];
        }
        *num_aggs = na;
    }
    free(S); free(tent);
    return rc;
}

/* ---------------------------------------------------------------------------
 * Coarse graph A_c <- coarsen(A) (Alg. 4 setup): vertices =
 * aggregates; (a, b), a != b, is an edge iff some stored fine entry (u, v)
 * has labels[u] = a and labels[v] = b.  Rows sorted, deduplicated, no
 * self-loops (reading Q21).
 *
 * Two-call convention: c_rowptr int64[na+1] is always filled; c_colinds is
 * written only if cap >= nnz_c (else ORC_ERANGE-like -7 and *nnz_c set).
 * ------------------------------------------------------------------------- */
static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

int orc_coarsen(int64_t n, const int64_t* rowptr, const int32_t* colinds, const int32_t* labels,
                int64_t na, int64_t* c_rowptr, int32_t* c_colinds, int64_t cap, int64_t* nnz_c) {
    if (n < 0 || na < 0 || !labels || !c_rowptr || !nnz_c) return ORC_EINVAL;
    for (int64_t v = 0; v < n; v++)
        if (labels[v] < 0 || labels[v] >= na) return ORC_EINVAL;
    /* members of each aggregate */
    int64_t* mptr = (int64_t*)calloc((size_t)na + 2, sizeof(int64_t));
    int64_t* mem = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
    if (!mptr || !mem) { free(mptr); free(mem); return ORC_ENOMEM; }
    for (int64_t v = 0; v < n; v++) mptr[labels[v] + 1]++;
    for (int64_t a = 0; a < na; a++) mptr[a + 1] += mptr[a];
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * ((size_t)na + 1));
    if (!fill) { free(mptr); free(mem); return ORC_ENOMEM; }
    memcpy(fill, mptr, sizeof(int64_t) * (size_t)na);
    for (int64_t v = 0; v < n; v++) mem[fill[labels[v]]++] = v;
    free(fill);

    /* per aggregate: the set {labels[v] : u in a, v in adj(u)} \ {a}, sorted */
    int32_t* buf = NULL;
    size_t bufcap = 0;
    int64_t total = 0;
    int rc = ORC_OK;
    c_rowptr[0] = 0;
    for (int64_t a = 0; a < na; a++) {
        size_t len = 0;
        for (int64_t k = mptr[a]; k < mptr[a + 1]; k++) {
            int64_t u = mem[k];
            len += (size_t)(rowptr[u + 1] - rowptr[u]);
        }
        if (len > bufcap) {
            free(buf);
            bufcap = len * 2;
            buf = (int32_t*)malloc(sizeof(int32_t) * bufcap);
            if (!buf) { rc = ORC_ENOMEM; break; }
        }
        size_t m = 0;
        for (int64_t k = mptr[a]; k < mptr[a + 1]; k++) {
            int64_t u = mem[k];
            for (int64_t j = rowptr[u]; j < rowptr[u + 1]; j++) {
                int32_t lb = labels[colinds[j]];
                if (lb != a) buf[m++] = lb;
            }
        }
        if (m) qsort(buf, m, sizeof(int32_t), cmp_i32);
        size_t uq = 0;
        for (size_t i = 0; i < m; i++) {
            if (i > 0 && buf[i] == buf[i - 1]) continue;
            if (c_colinds && total + (int64_t)uq < cap) c_colinds[total + uq] = buf[i];
            uq++;
        }
        total += (int64_t)uq;
        c_rowptr[a + 1] = total;
    }
    free(buf);
    free(mptr);
    free(mem);
    if (rc != ORC_OK) return rc;
    *nnz_c = total;
    if (!c_colinds || cap < total) return -7;
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * Alg. 4 "Cluster Multicolor Gauss-Seidel" (§III-C).
 *
 * Setup line "colorsets <- color(A_c)": the paper colours the
 * coarse graph with a greedy colouring ("setup time is dominated by
 * greedy graph coloring") without fixing the algorithm; reading Q30: the
 * deterministic parallel greedy of Jones-Plassmann, priorities = the MIS-2
 * status words of iteration 0 (word(0, v), seed as given, b of this graph).
 * Round r: every uncoloured vertex whose word is smaller than the words of
 * all its uncoloured neighbours (as of the start of the round) takes the
 * smallest colour not used by an already coloured neighbour.  Diagonal
 * entries are ignored.  Plain loops in round order.
 * ------------------------------------------------------------------------- */
int orc_color_jp(int64_t n, const int64_t* rowptr, const int32_t* colinds, uint64_t seed, int32_t* color,
                 int32_t* ncolors) {
    if (n < 0 || !color || !ncolors) return ORC_EINVAL;
    const int b = orc_bits(n);
    uint64_t* w = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
    unsigned char* cand = (unsigned char*)malloc((size_t)n + 1);
    unsigned char* used = NULL;
    size_t used_cap = 0;
    if (!w || !cand) { free(w); free(cand); return ORC_ENOMEM; }
    for (int64_t v = 0; v < n; v++) {
        w[v] = orc_word(ORC_SCHEME_XORSTAR, 0, v, seed, b);
        color[v] = -1;
    }
    int64_t left = n;
    int32_t nc = 0;
    int rc = ORC_OK;
    while (left > 0) {
        /* candidates of this round, from the colouring at its start */
        for (int64_t v = 0; v < n; v++) {
            cand[v] = 0;
            if (color[v] >= 0) continue;
            int ok = 1;
            for (int64_t j = rowptr[v]; j < rowptr[v + 1] && ok; j++) {
                const int64_t u = colinds[j];
                if (u != v && color[u] < 0 && w[u] < w[v]) ok = 0;
            }
            cand[v] = (unsigned char)ok;
        }
        for (int64_t v = 0; v < n; v++) {
            if (!cand[v]) continue;
            const size_t deg = (size_t)(rowptr[v + 1] - rowptr[v]);
            if (deg + 2 > used_cap) {
                free(used);
                used_cap = 2 * deg + 2;
                used = (unsigned char*)malloc(used_cap);
                if (!used) { rc = ORC_ENOMEM; break; }
            }
            memset(used, 0, deg + 2);
            for (int64_t j = rowptr[v]; j < rowptr[v + 1]; j++) {
                const int64_t u = colinds[j];
                if (u != v && color[u] >= 0 && !cand[u] && (size_t)color[u] <= deg) used[color[u]] = 1;
            }
            int32_t c = 0;
            while (used[c]) c++;
            color[v] = c;
            if (c + 1 > nc) nc = c + 1;
            left--;
        }
        if (rc != ORC_OK) break;
    }
    free(w);
    free(cand);
    free(used);
    *ncolors = nc;
    return rc;
}

/* Alg. 4 apply and its symmetric form ("looping over the
 * colors twice: first forward and then backward ... the order of row updates
 * within each cluster are reversed during the backward loop").  Row i belongs
 * to cluster labels[i]; cluster a has colour ccolor[a].  For each colour (in
 * order), for each cluster of that colour (independent: any order), for each
 * row of the cluster in ascending (forward) / descending (backward) order:
 *     r = b_i - sum_j A_ij x_j        (stored column order)
 *     x_i = x_i + r / A_ii            (reading Q31: the standard GS update;
 *                                      P:349's literal "x_i <- r/A_ii" with r
 *                                      including the diagonal term double
 *                                      counts it)
 * direction: 0 symmetric (forward then backward), 1 forward, 2 backward;
 * `sweeps` repetitions.  A_ii must be present and nonzero (else EINVAL). */
int orc_cluster_sgs(int64_t n, const int64_t* rowptr, const int32_t* colinds, const double* vals,
                    const int32_t* labels, int64_t na, const int32_t* ccolor, int32_t ncolors, const double* b,
                    double* x, int sweeps, int direction) {
    if (n < 0 || na < 0 || ncolors < 0 || sweeps < 0 || direction < 0 || direction > 2) return ORC_EINVAL;
    double* diag = (double*)malloc(sizeof(double) * ((size_t)n + 1));
    int64_t* mptr = (int64_t*)calloc((size_t)na + 2, sizeof(int64_t));
    int64_t* mem = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
    if (!diag || !mptr || !mem) { free(diag); free(mptr); free(mem); return ORC_ENOMEM; }
    int rc = ORC_OK;
    for (int64_t i = 0; i < n && rc == ORC_OK; i++) {
        diag[i] = 0.0;
        for (int64_t j = rowptr[i]; j < rowptr[i + 1]; j++)
            if (colinds[j] == i) diag[i] = vals[j];
        if (diag[i] == 0.0 || labels[i] < 0 || labels[i] >= na) rc = ORC_EINVAL;
    }
    /* rows of each cluster, ascending */
    if (rc == ORC_OK) {
        for (int64_t i = 0; i < n; i++) mptr[labels[i] + 1]++;
        for (int64_t a = 0; a < na; a++) mptr[a + 1] += mptr[a];
        int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * ((size_t)na + 1));
        if (!fill) rc = ORC_ENOMEM;
        else {
            memcpy(fill, mptr, sizeof(int64_t) * (size_t)na);
            for (int64_t i = 0; i < n; i++) mem[fill[labels[i]]++] = i;
            free(fill);
        }
    }
    for (int s = 0; s < sweeps && rc == ORC_OK; s++) {
        for (int pass = 0; pass < 2; pass++) {
            const int backward = (direction == 2) || (direction == 0 && pass == 1);
            if (direction == 1 && pass == 1) break;
            if (direction == 2 && pass == 1) break;
            for (int32_t ci = 0; ci < ncolors; ci++) {
                const int32_t col = backward ? ncolors - 1 - ci : ci;
                for (int64_t a = 0; a < na; a++) {
                    if (ccolor[a] != col) continue;
                    const int64_t k0 = mptr[a], k1 = mptr[a + 1];
                    for (int64_t t = 0; t < k1 - k0; t++) {
                        const int64_t i = mem[backward ? k1 - 1 - t : k0 + t];
                        double r = b[i];
                        for (int64_t j = rowptr[i]; j < rowptr[i + 1]; j++) r -= vals[j] * x[colinds[j]];
                        x[i] = x[i] + r / diag[i];
                    }
                }
            }
        }
    }
    free(diag);
    free(mptr);
    free(mem);
    return rc;
}

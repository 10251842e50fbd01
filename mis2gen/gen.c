/*
 * mis2gen/gen.c -- seeded synthetic CSR graph generators.
 *
 * This module is shared input infrastructure: it is used by BOTH the oracle
 * tests and the CUDA path's tests/bench, and therefore holds NONE of the
 * method's arithmetic (no hash, no status packing, no min-reductions).  It
 * only builds graphs shaped like the paper's workloads:
 *
 *   - 3-D (and 2-D, nz = 1) 7-point and 27-point Laplacian patterns with the
 *     diagonal stored, lexicographic ids id = x + nx*(y + ny*z)
 *     ("Laplace3D_100 is a 100^3 grid with a 7-point stencil";
 *     DESIGN.md reading Q26 for the ordering).
 *   - the "Elasticity3D" pattern: 27-point stencil (x) dense dof x dof block,
 *     dof-interleaved id = dof*point + c ("27-point stencil and 3 degrees
 *     of freedom"; reading Q25 -- reproduces |V| = 648,000 and
 *     |E| = 50,757,768 of tab:matrices-times P:486 exactly at 60^3).
 *   - a Graph500-style Kronecker/RMAT graph (A,B,C = 0.57,0.19,0.19), made
 *     symmetric, self-loop free and duplicate free (reading Q27).
 *
 * Every row of every generated graph is sorted ascending and duplicate free.
 * rowptr is int64[n+1], colinds is int32[nnz].
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- stencils */

static inline int in_range(int64_t a, int64_t n) { return a >= 0 && a < n; }

/* Number of valid stencil points (incl. the centre) around grid point (x,y,z). */
static inline int64_t stencil_count(int64_t x, int64_t y, int64_t z, int64_t nx, int64_t ny,
                                    int64_t nz, int kind) {
    if (kind == 7) {
        int64_t c = 1;
        c += (x > 0) + (x < nx - 1);
        c += (y > 0) + (y < ny - 1);
        c += (z > 0) + (z < nz - 1);
        return c;
    }
    /* 27-point: product of the per-axis extents */
    int64_t cx = 1 + (x > 0) + (x < nx - 1);
    int64_t cy = 1 + (y > 0) + (y < ny - 1);
    int64_t cz = 1 + (z > 0) + (z < nz - 1);
    return cx * cy * cz;
}

/* Total stored entries of the stencil (x) dof pattern, diagonal included. */
int64_t gen_stencil_nnz(int64_t nx, int64_t ny, int64_t nz, int kind, int dof) {
    if (nx < 1 || ny < 1 || nz < 1 || (kind != 7 && kind != 27) || dof < 1) return -1;
    int64_t pts = 0;
    #pragma omp parallel for reduction(+:pts) schedule(static)
    for (int64_t z = 0; z < nz; z++)
        for (int64_t y = 0; y < ny; y++)
            for (int64_t x = 0; x < nx; x++) pts += stencil_count(x, y, z, nx, ny, nz, kind);
    return pts * (int64_t)dof * (int64_t)dof;
}

/* Fill rowptr[n+1] and colinds[nnz]; n = nx*ny*nz*dof.  Returns nnz or -1. */
int64_t gen_stencil(int64_t nx, int64_t ny, int64_t nz, int kind, int dof, int64_t* rowptr,
                    int32_t* colinds) {
    if (nx < 1 || ny < 1 || nz < 1 || (kind != 7 && kind != 27) || dof < 1) return -1;
    const int64_t npts = nx * ny * nz;
    const int64_t n = npts * dof;
    /* row lengths */
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < npts; p++) {
        int64_t x = p % nx, y = (p / nx) % ny, z = p / (nx * ny);
        int64_t len = stencil_count(x, y, z, nx, ny, nz, kind) * dof;
        for (int c = 0; c < dof; c++) rowptr[p * dof + c + 1] = len;
    }
    rowptr[0] = 0;
    for (int64_t i = 0; i < n; i++) rowptr[i + 1] += rowptr[i];
    /* entries, ascending because (dz,dy,dx) ascend lexicographically and ids
     * are x-fastest, and the dof components ascend inside a point */
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < npts; p++) {
        int64_t x = p % nx, y = (p / nx) % ny, z = p / (nx * ny);
        for (int c = 0; c < dof; c++) {
            int64_t k = rowptr[p * dof + c];
            for (int dz = -1; dz <= 1; dz++)
                for (int dy = -1; dy <= 1; dy++)
                    for (int dx = -1; dx <= 1; dx++) {
                        int nzero = (dx != 0) + (dy != 0) + (dz != 0);
                        if (kind == 7 && nzero > 1) continue;
                        int64_t qx = x + dx, qy = y + dy, qz = z + dz;
                        if (!in_range(qx, nx) || !in_range(qy, ny) || !in_range(qz, nz)) continue;
                        int64_t q = qx + nx * (qy + ny * qz);
                        for (int c2 = 0; c2 < dof; c2++) colinds[k++] = (int32_t)(q * dof + c2);
                    }
        }
    }
    return rowptr[n];
}

/* --------------------------------------------------------------- Kronecker */

/* splitmix64: counter-based generator for the input recipe (not the method's
 * hash -- the method's priorities are xorshift*, implemented separately by the
 * oracle and by the CUDA path). */
static inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}
static inline double u01(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/*
 * Graph500-style Kronecker graph, n = 2^scale, m = edgefactor * n edge draws.
 *   edge e, level l: r = U[0,1) from splitmix64(seed, e, l); quadrant
 *   (0,0) w.p. A, (0,1) w.p. B, (1,0) w.p. C, (1,1) w.p. D = 1-A-B-C.
 * Vertex labels are permuted with a seeded Fisher-Yates shuffle.  Self-loops
 * dropped, each edge stored in both directions, duplicates removed, rows
 * sorted.  No diagonal is stored.
 *
 * Buffers: rowptr int64[n+1]; colbuf int32[2*m] (output occupies the first
 * nnz entries); eu, ev int32[m] scratch.  Returns nnz.
 */
int64_t gen_kronecker(int scale, int edgefactor, uint64_t seed, double A, double B, double C,
                      int64_t* rowptr, int32_t* colbuf, int32_t* eu, int32_t* ev) {
    if (scale < 1 || scale > 30 || edgefactor < 1) return -1;
    const int64_t n = (int64_t)1 << scale;
    const int64_t m = (int64_t)edgefactor * n;
    const double ab = A + B, abc = A + B + C;

    /* 1. seeded permutation of the labels */
    int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * n);
    if (!perm) return -2;
    for (int64_t i = 0; i < n; i++) perm[i] = (int32_t)i;
    uint64_t st = splitmix64(seed ^ 0x5eedULL);
    for (int64_t i = n - 1; i > 0; i--) {
        st = splitmix64(st);
        int64_t j = (int64_t)(st % (uint64_t)(i + 1));
        int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }

    /* 2. edge draws */
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; e++) {
        uint64_t u = 0, v = 0;
        uint64_t base = splitmix64(seed + 0x1000003ULL * (uint64_t)e);
        for (int l = 0; l < scale; l++) {
            double r = u01(splitmix64(base + (uint64_t)l));
            uint64_t bu, bv;
            if (r < A) { bu = 0; bv = 0; }
            else if (r < ab) { bu = 0; bv = 1; }
            else if (r < abc) { bu = 1; bv = 0; }
            else { bu = 1; bv = 1; }
            u |= bu << l; v |= bv << l;
        }
        eu[e] = perm[u];
        ev[e] = perm[v];
    }
    free(perm);

    /* 3. degree count (both directions, no self-loops) */
    int64_t* deg = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    if (!deg) return -2;
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; e++) {
        if (eu[e] == ev[e]) continue;
        #pragma omp atomic
        deg[eu[e]]++;
        #pragma omp atomic
        deg[ev[e]]++;
    }
    int64_t* start = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
    if (!start) { free(deg); return -2; }
    start[0] = 0;
    for (int64_t i = 0; i < n; i++) start[i + 1] = start[i] + deg[i];
    memset(deg, 0, sizeof(int64_t) * (size_t)n);
    /* 4. fill (order inside a row is scheduling dependent; fixed by the sort) */
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; e++) {
        int32_t a = eu[e], b = ev[e];
        if (a == b) continue;
        int64_t pa, pb;
        #pragma omp atomic capture
        pa = deg[a]++;
        #pragma omp atomic capture
        pb = deg[b]++;
        colbuf[start[a] + pa] = b;
        colbuf[start[b] + pb] = a;
    }
    /* 5. sort + dedupe rows, new lengths into deg */
    #pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; i++) {
        int32_t* r = colbuf + start[i];
        int64_t len = start[i + 1] - start[i];
        qsort(r, (size_t)len, sizeof(int32_t), cmp_i32);
        int64_t k = 0;
        for (int64_t j = 0; j < len; j++)
            if (k == 0 || r[j] != r[k - 1]) r[k++] = r[j];
        deg[i] = k;
    }
    /* 6. compact rows in order (destinations never overtake sources) */
    rowptr[0] = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t len = deg[i];
        if (rowptr[i] != start[i]) memmove(colbuf + rowptr[i], colbuf + start[i], sizeof(int32_t) * (size_t)len);
        rowptr[i + 1] = rowptr[i] + len;
    }
    free(start);
    free(deg);
    return rowptr[n];
}

/* ------------------------------------------------------------------ misc */

/* FNV-1a 64 over the bytes of rowptr and colinds (input checksum). */
uint64_t gen_checksum(int64_t n, const int64_t* rowptr, const int32_t* colinds) {
    uint64_t h = 0xcbf29ce484222325ULL;
    const unsigned char* p = (const unsigned char*)rowptr;
    for (int64_t i = 0; i < (n + 1) * 8; i++) { h ^= p[i]; h *= 0x100000001b3ULL; }
    p = (const unsigned char*)colinds;
    int64_t nb = rowptr[n] * 4;
    for (int64_t i = 0; i < nb; i++) { h ^= p[i]; h *= 0x100000001b3ULL; }
    return h;
}

int gen_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Brick-DDA equivalence check (tools only, not shipped).
 *
 * Restates, on the CPU, the traversal the GPU kernels use below brick level
 * bl = max(0, depth - 3): the reference's node-by-node descent
 * (kernels.py:600-647) down to level bl, then an exact voxel DDA across the
 * brick's n^3 leaf cells (n = 2^(depth - bl)) driven by a per-brick
 * occupancy table.  Writes the same (leaf, t0, t1) segments as
 * collect_segments_kernel (kernels.py:338-367) so tests/tools can compare
 * them bit for bit with the oracle, and counts the work (node steps, brick
 * entries, DDA steps) per ray.
 *
 *   gcc -O2 -shared -fPIC -ffp-contract=off -o tools/_build/libbrick_dda.so tools/brick_dda_check.c
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline double py_max(double a, double b) { return (b > a) ? b : a; }
static inline double py_min(double a, double b) { return (b < a) ? b : a; }

typedef struct {
    int depth, bl, n;       /* brick level, cells per brick axis */
    int64_t lo, count;      /* brick nodes are ptr in [lo, lo + count) */
    uint32_t *mask;         /* (count, 16) occupancy words, cell = x + 8y + 64z */
    uint32_t *base;         /* (count, 16) perm offset of the word's first leaf */
    int32_t *perm;          /* leaves in brick-cell order */
} bricks;

static void fill(const int32_t *child, int depth, int64_t ptr, int level, int x, int y, int z, int32_t *cell_leaf) {
    if (level == depth) {
        cell_leaf[x + 8 * y + 64 * z] = (int32_t)ptr;
        return;
    }
    for (int c = 0; c < 8; ++c) {
        int32_t p = child[ptr * 8 + c];
        if (p >= 0) fill(child, depth, p, level + 1, 2 * x + (c & 1), 2 * y + ((c >> 1) & 1), 2 * z + ((c >> 2) & 1), cell_leaf);
    }
}

/* frontier walk from the root down to level bl; returns a heap bricks* */
void *bdc_build(const int32_t *child, int64_t n_internal, int depth, int64_t n_leaves) {
    bricks *b = (bricks *)calloc(1, sizeof(bricks));
    b->depth = depth;
    b->bl = depth > 3 ? depth - 3 : 0;
    b->n = 1 << (depth - b->bl);
    int64_t *front = (int64_t *)malloc(sizeof(int64_t) * (n_internal + 1));
    int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (n_internal + 1));
    int64_t nf = 1;
    front[0] = 0;
    for (int L = 0; L < b->bl; ++L) {
        int64_t nn = 0;
        for (int64_t i = 0; i < nf; ++i)
            for (int c = 0; c < 8; ++c) {
                int32_t p = child[front[i] * 8 + c];
                if (p >= 0) next[nn++] = p;
            }
        int64_t *t = front; front = next; next = t; nf = nn;
    }
    int64_t lo = INT64_MAX, hi = -1;
    for (int64_t i = 0; i < nf; ++i) {
        if (front[i] < lo) lo = front[i];
        if (front[i] > hi) hi = front[i];
    }
    if (nf == 0) lo = hi = 0;
    b->lo = lo;
    b->count = hi - lo + 1;
    b->mask = (uint32_t *)calloc((size_t)b->count * 16, 4);
    b->base = (uint32_t *)calloc((size_t)b->count * 16, 4);
    b->perm = (int32_t *)malloc(sizeof(int32_t) * (n_leaves + 1));
    int32_t cell_leaf[512];
    int64_t off = 0;
    for (int64_t i = 0; i < nf; ++i) {
        for (int c = 0; c < 512; ++c) cell_leaf[c] = -1;
        if (depth == b->bl) cell_leaf[0] = (int32_t)front[i]; /* not reachable: bl < depth */
        else fill(child, depth, front[i], b->bl, 0, 0, 0, cell_leaf);
        int64_t bi = front[i] - lo;
        for (int w = 0; w < 16; ++w) {
            b->base[bi * 16 + w] = (uint32_t)off;
            uint32_t m = 0;
            for (int k = 0; k < 32; ++k)
                if (cell_leaf[32 * w + k] >= 0) {
                    m |= 1u << k;
                    b->perm[off++] = cell_leaf[32 * w + k];
                }
            b->mask[bi * 16 + w] = m;
        }
    }
    free(front);
    free(next);
    return b;
}

void bdc_free(void *p) {
    bricks *b = (bricks *)p;
    free(b->mask); free(b->base); free(b->perm); free(b);
}

typedef struct { int64_t ptr; int level; int64_t cx, cy, cz; double tin, tout; } ent;

/* one ray; mirrors collect_one of the oracle above brick level */
static int64_t ray_dda(const int32_t *child, const bricks *B, const double *o_, const double *d_, const double *lo,
                       double side, double tmin, double tmax, int64_t *leaf_out, double *t0_out, double *t1_out,
                       int64_t cap, int64_t *work, int64_t limit) {
    double o0 = (o_[0] - lo[0]) / side, o1 = (o_[1] - lo[1]) / side, o2 = (o_[2] - lo[2]) / side;
    double d0 = d_[0] / side, d1 = d_[1] / side, d2 = d_[2] / side;
    int mirror = 0;
    if (d0 < 0.0) { o0 = 1.0 - o0; d0 = -d0; mirror |= 1; }
    if (d1 < 0.0) { o1 = 1.0 - o1; d1 = -d1; mirror |= 2; }
    if (d2 < 0.0) { o2 = 1.0 - o2; d2 = -d2; mirror |= 4; }
    int ok = 1;
    double i0, i1, i2;
    if (d0 < 1e-300) { if (o0 < 0.0 || o0 >= 1.0) ok = 0; i0 = 1e300; } else i0 = 1.0 / d0;
    if (d1 < 1e-300) { if (o1 < 0.0 || o1 >= 1.0) ok = 0; i1 = 1e300; } else i1 = 1.0 / d1;
    if (d2 < 1e-300) { if (o2 < 0.0 || o2 >= 1.0) ok = 0; i2 = 1e300; } else i2 = 1.0 / d2;
    if (!ok) return 0;
    double rt_in = py_max(py_max((0.0 - o0) * i0, (0.0 - o1) * i1), py_max((0.0 - o2) * i2, tmin));
    double rt_out = py_min(py_min((1.0 - o0) * i0, (1.0 - o1) * i1), py_min((1.0 - o2) * i2, tmax));
    if (!(rt_in < rt_out)) return 0;
    ent st[256];
    int top = 0;
    st[top++] = (ent){0, 0, 0, 0, 0, rt_in, rt_out};
    int64_t count = 0;
    const int n = B->n;
    while (top > 0) {
        ent e = st[--top];
        if (e.level == B->bl) {
            /* ---- brick: exact DDA over n^3 leaf cells */
            work[1]++;
            const double hb = 1.0 / (double)((int64_t)1 << e.level), h = hb / n;
            const double xl = (double)e.cx * hb, yl = (double)e.cy * hb, zl = (double)e.cz * hb;
            const double tin = e.tin, tout = e.tout;
            int ix = 0, iy = 0, iz = 0;
            for (int s = n / 2; s >= 1; s /= 2) {
                if (((xl + (double)(ix + s) * h) - o0) * i0 < tin) ix += s;
                if (((yl + (double)(iy + s) * h) - o1) * i1 < tin) iy += s;
                if (((zl + (double)(iz + s) * h) - o2) * i2 < tin) iz += s;
            }
            double px = xl + (double)(ix + 1) * h, py = yl + (double)(iy + 1) * h, pz = zl + (double)(iz + 1) * h;
            double tx = (px - o0) * i0, ty = (py - o1) * i1, tz = (pz - o2) * i2;
            double tc = tin;
            const int64_t bi = e.ptr - B->lo;
            const int mx = (mirror & 1) ? n - 1 : 0, my = (mirror & 2) ? n - 1 : 0, mz = (mirror & 4) ? n - 1 : 0;
            for (;;) {
                work[2]++;
                double to = py_min(py_min(tx, ty), py_min(tz, tout));
                if (to > tc) {
                    int cell = (ix ^ mx) + 8 * (iy ^ my) + 64 * (iz ^ mz);
                    uint32_t m = B->mask[bi * 16 + (cell >> 5)];
                    uint32_t bit = 1u << (cell & 31);
                    if (m & bit) {
                        int64_t L = B->perm[B->base[bi * 16 + (cell >> 5)] + __builtin_popcount(m & (bit - 1))];
                        if (leaf_out && count < cap) {
                            leaf_out[count] = L;
                            t0_out[count] = tc;
                            t1_out[count] = to;
                        }
                        ++count;
                        if (count == limit) return count;
                    }
                }
                if (to >= tout) break;
                if (tx <= ty && tx <= tz) { ++ix; px = px + h; tx = (px - o0) * i0; }
                else if (ty <= tz) { ++iy; py = py + h; ty = (py - o1) * i1; }
                else { ++iz; pz = pz + h; tz = (pz - o2) * i2; }
                tc = to;
            }
            continue;
        }
        if (e.level == B->depth) { /* leaf (only when bl == depth, unused) */
            ++count;
            continue;
        }
        /* ---- node step (kernels.py:600-647) */
        work[0]++;
        ent c[8];
        int nc = 0;
        double h = 1.0 / (double)((int64_t)1 << (e.level + 1));
        double txm = ((double)(2 * e.cx + 1) * h - o0) * i0;
        double tym = ((double)(2 * e.cy + 1) * h - o1) * i1;
        double tzm = ((double)(2 * e.cz + 1) * h - o2) * i2;
        int b = 0;
        if (txm < e.tin) b |= 1;
        if (tym < e.tin) b |= 2;
        if (tzm < e.tin) b |= 4;
        double tin = e.tin;
        for (;;) {
            double tx = !(b & 1) ? txm : 1e301, ty = !(b & 2) ? tym : 1e301, tz = !(b & 4) ? tzm : 1e301;
            double to = py_min(py_min(tx, ty), py_min(tz, e.tout));
            int32_t cptr = child[e.ptr * 8 + (b ^ mirror)];
            if (cptr >= 0 && to > tin)
                c[nc++] = (ent){cptr, e.level + 1, 2 * e.cx + (b & 1), 2 * e.cy + ((b >> 1) & 1),
                                2 * e.cz + ((b >> 2) & 1), tin, to};
            if (to >= e.tout) break;
            if (tx <= ty && tx <= tz) b |= 1;
            else if (ty <= tz) b |= 2;
            else b |= 4;
            tin = to;
        }
        for (int a = nc - 1; a >= 0; --a) st[top++] = c[a];
    }
    return count;
}

/* segments per ray into CSR slots (ray_start from the oracle's counts);
 * work: (n, 3) node steps, brick entries, DDA steps */
int bdc_collect(const int32_t *child, void *bp, const double *lo, double side, const double *origins,
                const double *dirs, int64_t n, double tmin, double tmax, const int64_t *ray_start, int64_t *seg_leaf,
                double *seg_t0, double *seg_t1, int64_t *counts, int64_t *work, const int64_t *limit) {
    const bricks *B = (const bricks *)bp;
    for (int64_t r = 0; r < n; ++r) {
        int64_t b = ray_start ? ray_start[r] : 0, cap = ray_start ? ray_start[r + 1] - b : 0;
        work[3 * r] = work[3 * r + 1] = work[3 * r + 2] = 0;
        counts[r] = ray_dda(child, B, origins + 3 * r, dirs + 3 * r, lo, side, tmin, tmax,
                            ray_start ? seg_leaf + b : NULL, seg_t0 ? seg_t0 + b : NULL, seg_t1 ? seg_t1 + b : NULL,
                            cap, work + 3 * r, limit ? limit[r] : -1);
    }
    return 0;
}

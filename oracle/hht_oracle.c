/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the hierarchical slope-intercept Hough
 * transform of Singh & Bhatia, arXiv 1007.0547 ("A fast decision technique for hierarchical
 * Hough transform for line detection"), removal off. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this file's library. It shares no code,
 * header, table or constant with the CUDA path in paper_1007_0547_b200/csrc/, and neither side
 * includes or links the other.
 *
 * Everything is integer (int64), following the paper's own precision claim ("we do not undergo
 * any floating point operation", §4.3). Each function cites the passage it restates.
 *
 * Geometry (DESIGN.md §2 readings R1-R4):
 *   - an edge point (x0,y0) maps to the parameter-space line b = y0 - x0*m   (§1);
 *     for the BETA set the point is taken as (y0,x0)                         (§3);
 *   - the root region is m in [-1,1] x b in [-N,2N]  (reading R1; |m|<=1 from PAPER.md:25,67);
 *   - level l splits the root into 2^l x 2^l equal squares; level D is the leaf level
 *     ("at level ceil(log2 N)"); corners lie on the lattice
 *        m_i = -1 + 2*i/2^D,   b_j = -N + 3N*j/2^D,   i,j in [0, 2^D];
 *     a level-l region (a,c) has SW corner (a*s, c*s) and side s = 2^(D-l) lattice steps;
 *   - corner (m_c,b_c) is "above the line" when F = b_c - (-x0)*m_c - y0 >= 0, i.e. the paper's
 *     F(x0,y0) = y0 - m*x0 - b >= 0 (§2) written for a point (m_c,b_c) against the
 *     line with slope -x0 and intercept y0; otherwise it is "below" and its bit is 1
 *     ("A bit is 1, if the corner point is below the line");
 *   - bit order NE, NW, SW, SE, NE leftmost (getcode() PAPER.md:148-164);
 *   - a line votes for a region iff code != 0000 and code != 1111 (step 5;
 *     PAPER.md:115-118, step 12.b.v);
 *   - a region with votes > THRESHOLD is subdivided (PAPER.md:122 step 13, reading R5: strict,
 *     also at the root), children visited NE, NW, SW, SE, each child testing
 *     only the lines that voted for its parent (PAPER.md:100-103 step 12.b); a leaf-level region
 *     with votes > THRESHOLD is a solution; solution()'s point removal is OFF
 *     (reading R7).
 *
 * Scaled integer form of the corner test (multiply F by 2^D > 0, sign unchanged):
 *     2^D*m_c = -2^D + 2i,  2^D*b_c = -N*2^D + 3N*j,
 *     below  <=>  F < 0  <=>  2^D*b_c + x0*(2^D*m_c) - 2^D*y0 < 0.
 *
 * Parity pins: tests/test_oracle_pins.py (SPEC worked examples, Fig. 2 prose example, exact
 * rational cross-check, brute force, invariants, survey worked example; both circumcircle variants
 * against the minimised point-to-line distance in exact rationals, the horizontal-line closed form
 * and the survey's L9 totals). scripts/mutate_oracle.py: every listed mutant fails a pin.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_ALPHA 1
#define ORACLE_BETA 2
#define ORACLE_MAXLEV 64

/* ------------------------------------------------------------------------------------------ */
/* Corner test and 4-bit code                                                                  */
/* ------------------------------------------------------------------------------------------ */

/* Effective point of a half: ALPHA uses (x,y), BETA uses (y,x). */
static void effective_point(int32_t x, int32_t y, int half, int64_t *ex, int64_t *ey) {
    if (half == ORACLE_BETA) { *ex = y; *ey = x; }
    else { *ex = x; *ey = y; }
}

/* 1 iff lattice corner (i,j) lies strictly below the line b = ey - ex*m. */
int oracle_corner_below(int64_t ex, int64_t ey, int32_t N, int32_t D, int64_t i, int64_t j) {
    const int64_t scale = (int64_t)1 << D;                 /* 2^D */
    const int64_t m_scaled = -scale + 2 * i;               /* 2^D * m_c */
    const int64_t b_scaled = -(int64_t)N * scale + 3 * (int64_t)N * j;   /* 2^D * b_c */
    const int64_t F_scaled = b_scaled + ex * m_scaled - scale * ey;      /* 2^D * F(m_c, b_c) */
    return F_scaled < 0;   /* F >= 0: above or on -> bit 0; F < 0: below -> bit 1 */
}

/* Assemble the 4-bit code from the corner bits in the paper's order: NE is bit 1 (leftmost,
 * value 8), NW bit 2 (4), SW bit 3 (2), SE bit 4 (1) -- getcode(). */
static int assemble_code(int ne, int nw, int sw, int se) {
    int code = 0;              /* "Code <- 0000" */
    if (ne) code |= 8;         /* "If NorthEast corner of the region is below the line then Bit 1 is set to 1" */
    if (nw) code |= 4;         /* NorthWest -> Bit 2 */
    if (sw) code |= 2;         /* SouthWest -> Bit 3 */
    if (se) code |= 1;         /* SouthEast -> Bit 4 */
    return code;
}

/* getcode() for a parameter-space region (level l, index (a,c)); East = +m, North = +b. */
int oracle_code(int32_t x, int32_t y, int32_t half, int32_t N, int32_t D, int32_t level,
                int64_t a, int64_t c) {
    int64_t ex, ey;
    effective_point(x, y, half, &ex, &ey);
    const int64_t s = (int64_t)1 << (D - level);
    const int64_t i0 = a * s, j0 = c * s;
    return assemble_code(oracle_corner_below(ex, ey, N, D, i0 + s, j0 + s),   /* NE */
                         oracle_corner_below(ex, ey, N, D, i0, j0 + s),       /* NW */
                         oracle_corner_below(ex, ey, N, D, i0, j0),           /* SW */
                         oracle_corner_below(ex, ey, N, D, i0 + s, j0));      /* SE */
}

/* Vote rule, "if code != 0000 and code != 1111 then vote". */
int oracle_votes_for(int code) { return code != 0 && code != 15; }

/* getcode() on a generic axis-aligned square [x0,x0+side] x [y0,y0+side] of the image plane
 * against the line y = m*x + b with m = m_num/m_den, b = b_num/b_den (m_den, b_den > 0):
 * corner (X,Y) is above iff F = Y - m*X - b >= 0, bit 1 iff below. Used to pin
 * the bit order and the above/below convention on the paper's Fig. 2 style examples. */
int oracle_generic_code(int64_t m_num, int64_t m_den, int64_t b_num, int64_t b_den,
                        int64_t x0, int64_t y0, int64_t side) {
    /* F * m_den * b_den = Y*m_den*b_den - m_num*X*b_den - b_num*m_den  (denominators > 0) */
#define F_BELOW(X, Y) (((Y) * m_den * b_den - m_num * (X) * b_den - b_num * m_den) < 0)
    int ne = F_BELOW(x0 + side, y0 + side);
    int nw = F_BELOW(x0, y0 + side);
    int sw = F_BELOW(x0, y0);
    int se = F_BELOW(x0 + side, y0);
#undef F_BELOW
    return assemble_code(ne, nw, sw, se);
}

/* FHT [9]-style membership ("calculates the perpendicular distance to the line from
 * the center of the region and compares it with the radius of the circle circumscribing the
 * region"). Distances are measured in lattice units (the region is an s x s square,
 * SPEC.md:258 reading). With the line written as L(i,j) = 2^D*(ex+ey+N) - 2*ex*i - 3N*j = 0
 * (the negated scaled F above), distance(centre) <= circumradius s/sqrt(2) becomes, exactly in
 * integers, (2*L(centre))^2 <= 2*s^2*((2ex)^2 + (3N)^2), with 2*L(centre) = L evaluated at the
 * doubled centre coordinates (2*i0+s, 2*j0+s). */
int oracle_circle_passes(int32_t x, int32_t y, int32_t half, int32_t N, int32_t D, int32_t level,
                         int64_t a, int64_t c) {
    int64_t ex, ey;
    effective_point(x, y, half, &ex, &ey);
    const int64_t s = (int64_t)1 << (D - level);
    const int64_t i2 = 2 * a * s + s, j2 = 2 * c * s + s;             /* doubled centre */
    const __int128 L2 = (__int128)2 * (((int64_t)1 << D) * (ex + ey + N)) - 2 * ex * i2 - 3 * (int64_t)N * j2;
    const __int128 lhs = L2 * L2;
    const __int128 rhs = (__int128)2 * s * s * (4 * ex * ex + 9 * (int64_t)N * N);
    return lhs <= rhs;
}

/* The same FHT [9]-style test with the distance and the circumradius measured in
 * the (m, b) units of the parameter space itself (reading R22): a level-l region is
 * the rectangle of width w = 2s/2^D (in m) and height h = 3N*s/2^D (in b), its circumcircle has
 * radius sqrt(w^2 + h^2)/2, and the line b + ex*m - ey = 0 lies at distance |F(centre)|/sqrt(1+ex^2)
 * from the centre, F(m, b) = b + ex*m - ey (the negated F of PAPER.md:51). Squared and multiplied by
 * 4^(D+1) > 0:  (2^(D+1) F(centre))^2 <= (1 + ex^2) * (4 s^2 + 9 N^2 s^2), where 2^(D+1)*F(centre) is
 * exact in integers at the doubled centre (2*i0+s, 2*j0+s):
 *     2^(D+1) m_c = -2^(D+1) + 2*i2,  2^(D+1) b_c = -N*2^(D+1) + 3N*j2.
 * Exact in __int128 while (1 + N^2) * 4^D * (4 + 9 N^2) < 2^127 (N <= 2^16 and D <= 24). */
int oracle_circle_mb_passes(int32_t x, int32_t y, int32_t half, int32_t N, int32_t D, int32_t level,
                            int64_t a, int64_t c) {
    int64_t ex, ey;
    effective_point(x, y, half, &ex, &ey);
    const int64_t s = (int64_t)1 << (D - level);
    const int64_t i2 = 2 * a * s + s, j2 = 2 * c * s + s;             /* doubled centre */
    const __int128 sc = (__int128)1 << (D + 1);                        /* 2^(D+1) */
    const __int128 m2 = -sc + 2 * (__int128)i2;                        /* 2^(D+1) * m_c */
    const __int128 b2 = -(__int128)N * sc + 3 * (__int128)N * j2;      /* 2^(D+1) * b_c */
    const __int128 F2 = b2 + ex * m2 - sc * ey;                        /* 2^(D+1) * F(centre) */
    const __int128 lhs = F2 * F2;
    const __int128 rhs = (__int128)(1 + ex * ex) * s * s * (4 + 9 * (__int128)N * N);
    return lhs <= rhs;
}

static int member(int variant, int32_t x, int32_t y, int32_t half, int32_t N, int32_t D,
                  int32_t level, int64_t a, int64_t c) {
    if (variant == 1) return oracle_circle_passes(x, y, half, N, D, level, a, c);
    if (variant == 2) return oracle_circle_mb_passes(x, y, half, N, D, level, a, c);
    return oracle_votes_for(oracle_code(x, y, half, N, D, level, a, c));
}

/* votes(R) by brute force over ALL points (SPEC.md:316-324 dense_votes, any level). */
int64_t oracle_region_votes(const int32_t *pts, int64_t n, int32_t half, int32_t N, int32_t D,
                            int32_t level, int64_t a, int64_t c, int32_t variant) {
    int64_t v = 0;
    for (int64_t p = 0; p < n; ++p)
        v += member(variant, pts[2 * p], pts[2 * p + 1], half, N, D, level, a, c);
    return v;
}

/* The classic dense accumulator at level `level`: acc[c * 2^level + a]. */
void oracle_dense_votes(const int32_t *pts, int64_t n, int32_t half, int32_t N, int32_t D,
                        int32_t level, uint32_t *acc) {
    const int64_t side = (int64_t)1 << level;
    for (int64_t c = 0; c < side; ++c)
        for (int64_t a = 0; a < side; ++a)
            acc[c * side + a] = (uint32_t)oracle_region_votes(pts, n, half, N, D, level, a, c, 0);
}

/* ------------------------------------------------------------------------------------------ */
/* Recursive depth-first detector (removal off)                               */
/* ------------------------------------------------------------------------------------------ */

typedef struct { uint32_t *v; int64_t n, cap; } vec_u32;

static int vec_push(vec_u32 *x, uint32_t a) {
    if (x->n == x->cap) {
        int64_t nc = x->cap ? 2 * x->cap : 64;
        uint32_t *nv = (uint32_t *)realloc(x->v, (size_t)nc * sizeof(uint32_t));
        if (!nv) return -1;
        x->v = nv; x->cap = nc;
    }
    x->v[x->n++] = a;
    return 0;
}

typedef struct oracle_result {
    int32_t N, D, halves, variant;
    int64_t T;
    vec_u32 level[2][ORACLE_MAXLEV];  /* per half: (a, c, votes) triplets in DFS order */
    vec_u32 leaves;                   /* (half, i, j, votes) quadruplets in DFS order */
    int64_t tests, votes, max_tests;
    int64_t visited[2][ORACLE_MAXLEV], split[2][ORACLE_MAXLEV];
    int truncated, oom;
    uint8_t *removed;                 /* removal on: per point of the current half, 1 = removed */
    vec_u32 support;                  /* removal on: (emitted leaf index, point index) pairs */
} oracle_result;

typedef struct {
    const int32_t *pts;
    int32_t half;
    oracle_result *r;
} dfs_ctx;

/* visit(l, a, c, cand): SURVEY.md §8(c) "Algorithm the oracle follows". cand holds the indices
 * of the points whose line crossed the parent (all points at the root). */
static void visit(dfs_ctx *k, int32_t l, int64_t a, int64_t c, const int64_t *cand, int64_t ncand) {
    oracle_result *r = k->r;
    if (r->oom || r->truncated) return;
    if (r->max_tests > 0 && r->tests >= r->max_tests) { r->truncated = 1; return; }
    const int hi = k->half == ORACLE_BETA;
    int64_t *voters = (int64_t *)malloc((size_t)(ncand > 0 ? ncand : 1) * sizeof(int64_t));
    if (!voters) { r->oom = 1; return; }
    int64_t nv = 0;
    for (int64_t q = 0; q < ncand; ++q) {                  /* steps 2-5 / 12.a-b */
        const int64_t p = cand[q];
        if (r->removed && r->removed[p]) continue;         /* solution(): its codes were set to 0000 */
        if (member(r->variant, k->pts[2 * p], k->pts[2 * p + 1], k->half, r->N, r->D, l, a, c))
            voters[nv++] = p;                              /* level.vote <- level.vote + 1 */
    }
    r->tests += ncand;                                     /* one code evaluation per candidate */
    r->votes += nv;
    r->visited[hi][l] += 1;
    vec_u32 *rec = &r->level[hi][l];
    if (vec_push(rec, (uint32_t)a) || vec_push(rec, (uint32_t)c) || vec_push(rec, (uint32_t)nv)) r->oom = 1;
    if (nv > r->T) {                                       /* step 13: level.vote > THRESHOLD */
        if (l == r->D) {                                   /* leaf: solution() */
            const uint32_t li = (uint32_t)(r->leaves.n / 4);
            if (vec_push(&r->leaves, (uint32_t)k->half) || vec_push(&r->leaves, (uint32_t)a) ||
                vec_push(&r->leaves, (uint32_t)c) || vec_push(&r->leaves, (uint32_t)nv)) r->oom = 1;
            if (r->removed) {
                /* plot every edge point whose leaf code is mixed, then set its
                 * codes at all levels to 0000 ("exclude the edge point from further calculations") */
                for (int64_t q = 0; q < nv; ++q) {
                    r->removed[voters[q]] = 1;
                    if (vec_push(&r->support, li) || vec_push(&r->support, (uint32_t)voters[q])) r->oom = 1;
                }
            }
        } else {
            r->split[hi][l] += 1;
            /* quad1..quad4 = NE, NW, SW, SE: (da,dc) = (1,1),(0,1),(0,0),(1,0) */
            static const int da[4] = {1, 0, 0, 1}, dc[4] = {1, 1, 0, 0};
            for (int q = 0; q < 4; ++q)
                visit(k, l + 1, 2 * a + da[q], 2 * c + dc[q], voters, nv);
        }
    }
    free(voters);
}

oracle_result *oracle_detect(const int32_t *pts, int64_t n, int32_t N, int32_t D, int64_t T,
                             int32_t halves, int32_t variant, int64_t max_tests) {
    if (D < 0 || D >= ORACLE_MAXLEV - 1 || N < 1 || n < 0) return NULL;
    oracle_result *r = (oracle_result *)calloc(1, sizeof(oracle_result));
    if (!r) return NULL;
    r->N = N; r->D = D; r->T = T; r->halves = halves; r->variant = variant; r->max_tests = max_tests;
    int64_t *all = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!all) { free(r); return NULL; }
    for (int64_t p = 0; p < n; ++p) all[p] = p;
    /* "The algorithm first processes the set ... ALPHA and then ... BETA" */
    for (int32_t h = ORACLE_ALPHA; h <= ORACLE_BETA; ++h) {
        if (!(halves & h)) continue;
        dfs_ctx k = {pts, h, r};
        visit(&k, 0, 0, 0, all, n);
    }
    free(all);
    return r;
}

/* The same depth-first detector with solution()'s point removal ON (SPEC.md:307,
 * 341, 348, 350): a leaf whose live votes exceed THRESHOLD emits its voters, which then vote nowhere
 * else; votes are counted on live points at visit time, so later siblings see reduced votes. Each
 * tree (half) removes from its own copy of the points (reading R13: every point enters both trees). */
oracle_result *oracle_detect_removal(const int32_t *pts, int64_t n, int32_t N, int32_t D, int64_t T,
                                     int32_t halves) {
    if (D < 0 || D >= ORACLE_MAXLEV - 1 || N < 1 || n < 0) return NULL;
    oracle_result *r = (oracle_result *)calloc(1, sizeof(oracle_result));
    if (!r) return NULL;
    r->N = N; r->D = D; r->T = T; r->halves = halves; r->variant = 0;
    int64_t *all = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    r->removed = (uint8_t *)malloc((size_t)(n > 0 ? n : 1));
    if (!all || !r->removed) { free(all); free(r->removed); free(r); return NULL; }
    for (int64_t p = 0; p < n; ++p) all[p] = p;
    for (int32_t h = ORACLE_ALPHA; h <= ORACLE_BETA; ++h) {
        if (!(halves & h)) continue;
        memset(r->removed, 0, (size_t)(n > 0 ? n : 1));
        dfs_ctx k = {pts, h, r};
        visit(&k, 0, 0, 0, all, n);
    }
    free(all);
    return r;
}

int64_t oracle_result_support_count(const oracle_result *r) { return r->support.n / 2; }
void oracle_result_support(const oracle_result *r, uint32_t *out) {
    if (r->support.n) memcpy(out, r->support.v, (size_t)r->support.n * sizeof(uint32_t));
}

/* Run the same visit() from region (level, a, c) with ALL points as candidates. By containment
 * (a line crossing a child crosses its parent) the subtree's records equal those of the full
 * run; only the candidate count (tests) at the subtree root differs. Used by scripts that write
 * golden digests for large configs in parallel. */
oracle_result *oracle_detect_subtree(const int32_t *pts, int64_t n, int32_t N, int32_t D, int64_t T,
                                     int32_t half, int32_t level, int64_t a, int64_t c) {
    oracle_result *r = (oracle_result *)calloc(1, sizeof(oracle_result));
    if (!r) return NULL;
    r->N = N; r->D = D; r->T = T; r->halves = half; r->variant = 0;
    int64_t *all = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!all) { free(r); return NULL; }
    for (int64_t p = 0; p < n; ++p) all[p] = p;
    dfs_ctx k = {pts, half, r};
    visit(&k, level, a, c, all, n);
    free(all);
    return r;
}

int64_t oracle_result_level_count(const oracle_result *r, int32_t half, int32_t level) {
    return r->level[half == ORACLE_BETA][level].n / 3;
}
void oracle_result_level(const oracle_result *r, int32_t half, int32_t level, uint32_t *out) {
    const vec_u32 *v = &r->level[half == ORACLE_BETA][level];
    if (v->n) memcpy(out, v->v, (size_t)v->n * sizeof(uint32_t));
}
int64_t oracle_result_leaf_count(const oracle_result *r) { return r->leaves.n / 4; }
void oracle_result_leaves(const oracle_result *r, uint32_t *out) {
    if (r->leaves.n) memcpy(out, r->leaves.v, (size_t)r->leaves.n * sizeof(uint32_t));
}
/* out[0..5] = tests, votes, leaves, truncated, oom, depth; out[8+l] = visited[half0][l] ... */
void oracle_result_stats(const oracle_result *r, int64_t *out) {
    out[0] = r->tests; out[1] = r->votes; out[2] = r->leaves.n / 4;
    out[3] = r->truncated; out[4] = r->oom; out[5] = r->D;
    for (int h = 0; h < 2; ++h)
        for (int l = 0; l < ORACLE_MAXLEV; ++l) {
            out[8 + h * ORACLE_MAXLEV + l] = r->visited[h][l];
            out[8 + 2 * ORACLE_MAXLEV + h * ORACLE_MAXLEV + l] = r->split[h][l];
        }
}
void oracle_result_free(oracle_result *r) {
    if (!r) return;
    for (int h = 0; h < 2; ++h)
        for (int l = 0; l < ORACLE_MAXLEV; ++l) free(r->level[h][l].v);
    free(r->leaves.v);
    free(r->support.v);
    free(r->removed);
    free(r);
}

// Mid-size latency path: the whole level-synchronous traversal of a detection too large for one
// block (k_small) but whose lists stay small (up to kMidMaxS entries per level), as ONE cooperative
// kernel over the whole GPU with grid barriers between its phases, instead of ~30 launches and a host
// synchronisation per split (the multi-kernel path, hht_driver.cu).
//
// Method (identical outputs to the multi-kernel path and the oracle): per level l, for every split
// region R (frontier) and every line of R's candidate list, the four child codes from the exact test
// 0 < G_SW(child) <= s_c (2ex + 3N) ("code != 0000 and code != 1111"; SURVEY.md §0 L3/L4:
// child SW values g, g - P, g - Q, g - P - Q); a child with votes > T splits and
// receives the lines that cross it; level D children with votes > T are the
// detected lines. Per level:
//   S1  (grid over tiles of the 4F children) records, split flags, tile-local scans of (split count,
//       list entries, chunks); tile totals to global memory
//   S2  (grid) every block scans the tile totals, then writes the next frontier (or the leaves) and
//       each child's next-frontier index
//   W   (grid over 256-entry chunks of the level's lists) appends every line to the lists of the
//       split children it crosses and counts, for each such child, the four grandchildren the line
//       crosses (count-ahead: the next level's child votes, so no level is read twice)
// with one grid barrier after each phase. Level 0 (the roots, whose lists are the trees' points)
// starts with a count pass.
#include <cooperative_groups.h>

#include "hht_internal.h"

namespace hht {
namespace {
namespace cg = cooperative_groups;

template <typename I> struct MidUnsigned;
template <> struct MidUnsigned<int32_t> { using type = uint32_t; };
template <> struct MidUnsigned<int64_t> { using type = uint64_t; };

// 0 < v <= U as one unsigned compare of v - 1
template <typename I>
__device__ __forceinline__ uint32_t mid_cross(I v_minus_1, I U) {
    using UI = typename MidUnsigned<I>::type;
    return (UI)v_minus_1 < (UI)U ? 1u : 0u;
}

// inclusive warp scan of two 16-bit fields packed in a word (each field's total <= 32 * 8 = 256)
__device__ __forceinline__ uint32_t warp_incl16(uint32_t v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, d);
        if (lane >= d) v += t;
    }
    return v;
}

struct Tri { uint32_t f, s, c; };

// Exclusive block scan of (f, s, c); returns the block totals. s_w: 3 * (warps + 1) words.
__device__ Tri block_excl3(Tri x, Tri& excl, uint32_t* s_w) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    Tri inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t tf = __shfl_up_sync(0xFFFFFFFFu, inc.f, d);
        const uint32_t ts = __shfl_up_sync(0xFFFFFFFFu, inc.s, d);
        const uint32_t tc = __shfl_up_sync(0xFFFFFFFFu, inc.c, d);
        if (lane >= d) { inc.f += tf; inc.s += ts; inc.c += tc; }
    }
    if (lane == 31) { s_w[3 * wid] = inc.f; s_w[3 * wid + 1] = inc.s; s_w[3 * wid + 2] = inc.c; }
    __syncthreads();
    if (wid == 0) {
        Tri w = lane < nw ? Tri{s_w[3 * lane], s_w[3 * lane + 1], s_w[3 * lane + 2]} : Tri{0, 0, 0};
        Tri wi = w;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t tf = __shfl_up_sync(0xFFFFFFFFu, wi.f, d);
            const uint32_t ts = __shfl_up_sync(0xFFFFFFFFu, wi.s, d);
            const uint32_t tc = __shfl_up_sync(0xFFFFFFFFu, wi.c, d);
            if (lane >= d) { wi.f += tf; wi.s += ts; wi.c += tc; }
        }
        if (lane < nw) { s_w[3 * lane] = wi.f - w.f; s_w[3 * lane + 1] = wi.s - w.s; s_w[3 * lane + 2] = wi.c - w.c; }
        if (lane == 31) { s_w[3 * 32] = wi.f; s_w[3 * 32 + 1] = wi.s; s_w[3 * 32 + 2] = wi.c; }
    }
    __syncthreads();
    excl = {s_w[3 * wid] + inc.f - x.f, s_w[3 * wid + 1] + inc.s - x.s, s_w[3 * wid + 2] + inc.c - x.c};
    const Tri tot{s_w[3 * 32], s_w[3 * 32 + 1], s_w[3 * 32 + 2]};
    __syncthreads();
    return tot;
}

// Region descriptor of a frontier entry (two 16-byte words, one vector load each):
//   d0 = (tree | beta << 31, a, c, list start), d1 = (list length, chunk offset, -, -)
__device__ __forceinline__ void put_desc(uint4* fd, uint32_t g, uint32_t t, bool beta, uint32_t a, uint32_t c,
                                         uint32_t start, uint32_t len, uint32_t coff) {
    fd[2 * g] = make_uint4(t | (beta ? 0x80000000u : 0u), a, c, start);
    fd[2 * g + 1] = make_uint4(len, coff, 0u, 0u);
}

struct MidChunk {
    uint4 d0, d1;                 // descriptor of the chunk's region
    uint32_t r, k;                // region, chunk index within the region
};

__device__ __forceinline__ MidChunk mid_fetch(const MidArgs& A, int cur, uint32_t ch, uint32_t C) {
    MidChunk m;
    if (ch < C) {
        m.r = __ldg(A.chunkmap[cur] + ch);
        m.d0 = __ldg(A.fd[cur] + 2 * m.r);
        m.d1 = __ldg(A.fd[cur] + 2 * m.r + 1);
        m.k = ch - m.d1.y;
    } else {
        m.r = 0; m.k = 0;
        m.d0 = make_uint4(0, 0, 0, 0);
        m.d1 = make_uint4(0, 0, 0, 0);
    }
    return m;
}

__device__ __forceinline__ void mid_items(uint32_t (&p)[kItems], const uint32_t* list, const MidChunk& m, int lane) {
    const uint32_t base = m.k * kChunk, len = m.d1.x;
    const uint32_t* src = list + m.d0.w + base + lane;
#pragma unroll
    for (int it = 0; it < kItems; ++it) p[it] = base + lane + kWarp * it < len ? __ldg(src + kWarp * it) : 0u;
}

// One 256-entry chunk of region m.r at level l: COUNT (level 0 only) adds the 4 child votes; else
// appends to the split children's lists and counts their grandchildren (count-ahead).
template <typename I, bool COUNT>
__device__ __forceinline__ void mid_chunk(const MidArgs& A, int l, int cur, const MidChunk& m,
                                          const uint32_t (&p)[kItems], int lane, bool append) {
    const uint32_t a = m.d0.y, c = m.d0.z, len = m.d1.x, r = m.r;
    const bool beta = (m.d0.x >> 31) != 0;
    const int D = A.D, sh = D - l;
    const I N = (I)A.N;
    const I i0 = (I)a << sh, j0 = (I)c << sh;
    const I alpha = ((I)1 << D) - 2 * i0;
    const I beta_m1 = (N << D) - (I)3 * N * j0 - 1;
    const I Qc = ((I)3 * N) << (sh - 1);
    const uint32_t base = m.k * kChunk;
    uint32_t cm = 0;                               // child bits, 4 per item (q = NE, NW, SW, SE)
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const I ex = (I)(beta ? (p[it] & 0xFFFFu) : (p[it] >> 16));
        const I ey = (I)(beta ? (p[it] >> 16) : (p[it] & 0xFFFFu));
        I gm1 = ex * alpha + (ey << D) + beta_m1;              // G(SW corner of R) - 1
        if (base + lane + kWarp * it >= len) gm1 = (I)-1;
        const I Pc = ex << sh, Uc = Pc + Qc;
        const uint32_t b = mid_cross<I>(gm1 - Pc - Qc, Uc) | (mid_cross<I>(gm1 - Qc, Uc) << 1) |
                           (mid_cross<I>(gm1, Uc) << 2) | (mid_cross<I>(gm1 - Pc, Uc) << 3);
        cm |= b << (4 * it);
    }
    if (COUNT) {
        const uint32_t c0 = __popc(cm & 0x11111111u), c1 = __popc(cm & 0x22222222u);
        const uint32_t c2 = __popc(cm & 0x44444444u), c3 = __popc(cm & 0x88888888u);
        const uint32_t s02 = __reduce_add_sync(0xFFFFFFFFu, c0 | (c2 << 16));
        const uint32_t s13 = __reduce_add_sync(0xFFFFFFFFu, c1 | (c3 << 16));
        if (lane < 4) {
            const uint32_t v = lane == 0 ? (s02 & 0xFFFFu) : lane == 1 ? (s13 & 0xFFFFu) : lane == 2 ? (s02 >> 16) : (s13 >> 16);
            if (v) atomicAdd(A.cv[cur] + 4ull * r + lane, v);
        }
        return;
    }
    // split children: next-frontier index (kNone when the child is not split)
    const uint32_t my_f = lane < 4 ? A.cursor[4ull * r + lane] : kNone;
    uint32_t splitm = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) splitm |= (__shfl_sync(0xFFFFFFFFu, my_f, q) != kNone ? 1u : 0u) << q;
    cm &= splitm * 0x11111111u;
    if (__all_sync(0xFFFFFFFFu, cm == 0)) return;
    const uint32_t c0 = __popc(cm & 0x11111111u), c1 = __popc(cm & 0x22222222u);
    const uint32_t c2 = __popc(cm & 0x44444444u), c3 = __popc(cm & 0x88888888u);
    const uint32_t o02 = c0 | (c2 << 16), o13 = c1 | (c3 << 16);
    const uint32_t i02 = warp_incl16(o02, lane), i13 = warp_incl16(o13, lane);
    const uint32_t t02 = __shfl_sync(0xFFFFFFFFu, i02, 31), t13 = __shfl_sync(0xFFFFFFFFu, i13, 31);
    // reserve the runs first; the count-ahead below covers the atomics' round trip
    uint32_t my_base = 0;
    if (append && lane < 4 && my_f != kNone) {
        const uint32_t tq = lane == 0 ? (t02 & 0xFFFFu) : lane == 1 ? (t13 & 0xFFFFu) : lane == 2 ? (t02 >> 16) : (t13 >> 16);
        if (tq) my_base = __ldg(&A.fd[cur ^ 1][2 * my_f].w) + atomicAdd(A.app + my_f, tq);
    }
    // count-ahead: grandchild (q, qq) in 16-bit field (4q + qq) & 1 of word (4q + qq) >> 1
    uint32_t gw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const I ex = (I)(beta ? (p[it] & 0xFFFFu) : (p[it] >> 16));
        const I ey = (I)(beta ? (p[it] >> 16) : (p[it] & 0xFFFFu));
        const I gm1 = ex * alpha + (ey << D) + beta_m1;
        const I Pc = ex << sh;
        const I Pg = Pc >> 1, Qg = Qc >> 1, Ug = Pg + Qg;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!((cm >> (4 * it + q)) & 1u)) continue;
            const I gq = gm1 - (I)quad_da(q) * Pc - (I)quad_dc(q) * Qc;   // G(SW of child q) - 1
            const uint32_t b0 = mid_cross<I>(gq - Pg - Qg, Ug), b1 = mid_cross<I>(gq - Qg, Ug);
            const uint32_t b2 = mid_cross<I>(gq, Ug), b3 = mid_cross<I>(gq - Pg, Ug);
            gw[2 * q] += b0 | (b1 << 16);
            gw[2 * q + 1] += b2 | (b3 << 16);
        }
    }
    uint32_t sw = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const uint32_t s = __reduce_add_sync(0xFFFFFFFFu, gw[w]);
        if ((lane >> 1) == w) sw = s;
    }
    const uint32_t v = (sw >> (16 * (lane & 1))) & 0xFFFFu;
    const uint32_t fl = __shfl_sync(0xFFFFFFFFu, my_f, (lane >> 2) & 3);
    if (lane < 16 && fl != kNone && v) atomicAdd(A.cv[cur ^ 1] + 4ull * fl + (lane & 3), v);
    // append: per-lane runs at the reserved bases (not at level D-2: level D-1 lists are never read,
    // its children's votes are this count-ahead)
    if (!append) return;
    const uint32_t e02 = i02 - o02, e13 = i13 - o13;
    uint32_t pos[4];
    pos[0] = __shfl_sync(0xFFFFFFFFu, my_base, 0) + (e02 & 0xFFFFu);
    pos[1] = __shfl_sync(0xFFFFFFFFu, my_base, 1) + (e13 & 0xFFFFu);
    pos[2] = __shfl_sync(0xFFFFFFFFu, my_base, 2) + (e02 >> 16);
    pos[3] = __shfl_sync(0xFFFFFFFFu, my_base, 3) + (e13 >> 16);
    uint32_t* out = A.list[cur ^ 1];
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if ((cm >> (4 * it + q)) & 1u) out[pos[q]++] = p[it];
    }
}

// All chunks of one level, each warp walking chunks warp, warp + nwarps, ... with the next chunk's
// descriptor and entries in flight while the current one is processed.
template <typename I, bool COUNT>
__device__ __forceinline__ void mid_pass(const MidArgs& A, int l, int cur, uint32_t C, uint32_t warp, uint32_t nwarps,
                                         int lane, bool append) {
    const uint32_t* list = l == 0 ? A.packed : A.list[cur];
    uint32_t ch = warp;
    MidChunk m = mid_fetch(A, cur, ch, C);
    uint32_t p[kItems];
    mid_items(p, list, m, lane);
    for (; ch < C; ch += nwarps) {
        const MidChunk mn = mid_fetch(A, cur, ch + nwarps, C);
        uint32_t pn[kItems];
        mid_items(pn, list, mn, lane);
        mid_chunk<I, COUNT>(A, l, cur, m, p, lane, append);
        m = mn;
#pragma unroll
        for (int it = 0; it < kItems; ++it) p[it] = pn[it];
    }
}

template <typename I>
__global__ void __launch_bounds__(kMidThreads, kMidMinBlocks) k_mid(const MidArgs A) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t s_w[3 * 33];
    __shared__ uint32_t s_pref[3 * kMidMaxTiles];
    __shared__ unsigned long long s_acc[2];
    __shared__ uint32_t s_tot[3];
    const int lane = threadIdx.x & 31;
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gsize = (uint64_t)gridDim.x * blockDim.x;
    const uint32_t warp = (uint32_t)(gtid >> 5), nwarps = (uint32_t)(gsize >> 5);
    const int D = A.D;
    // ---- K0 in the same launch: stage and range-check the points; the flag is read after
    // the first grid barrier, and an out-of-range point ends the call before any traversal
    if (A.pts) {
        uint32_t bad = 0;
        for (uint64_t i = gtid; i < A.npts; i += gsize) {
            const int2 p = A.pts[i];
            const bool ok = (unsigned)p.x < (unsigned)A.N && (unsigned)p.y < (unsigned)A.N;
            bad |= !ok;
            A.packed[i] = ok ? (((uint32_t)p.x << 16) | (uint32_t)p.y) : 0u;
        }
        if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(A.ctl + 3, 1u);
    }
    // ---- level 0: the roots (every line crosses the root); split iff E > T (R6)
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < kStatCount; i += blockDim.x) A.stats[i] = 0;   // the call's statistics
        for (int i = threadIdx.x; i < D + 2; i += blockDim.x) A.counts[i] = 0;     // levels never reached stay 0
        __syncthreads();
        const uint32_t nt = A.ntrees;
        unsigned long long tests = 0, votes = 0;
        uint32_t carry_f = 0, carry_c = 0;
        for (uint32_t t0 = 0; t0 < nt; t0 += blockDim.x) {
            const uint32_t t = t0 + threadIdx.x;
            const uint32_t E = t < nt ? A.tree_n[t] : 0u;
            const bool split = t < nt && (uint64_t)E > A.T;
            if (t < nt) {
                A.rec[0][t] = {t, 0, 0, E};
                tests += E + (split ? 4ull * E : 0ull);
                votes += E;
            }
            Tri ex;
            const Tri tot = block_excl3(Tri{split ? 1u : 0u, 0u, split ? (E + kChunk - 1) / kChunk : 0u}, ex, s_w);
            if (split) {
                const uint32_t f = carry_f + ex.f, co = carry_c + ex.c;
                put_desc(A.fd[0], f, t, A.tree_beta[t] != 0, 0, 0, (uint32_t)A.tree_off[t], E, co);
                A.cv[0][4 * f] = 0; A.cv[0][4 * f + 1] = 0; A.cv[0][4 * f + 2] = 0; A.cv[0][4 * f + 3] = 0;
                for (uint32_t q = 0, nc = (E + kChunk - 1) / kChunk; q < nc; ++q) A.chunkmap[0][co + q] = f;
            }
            carry_f += tot.f;
            carry_c += tot.c;
        }
        if (threadIdx.x == 0) { A.ctl[0] = carry_f; A.ctl[1] = carry_c; }
        atomicAdd(A.stats + kStatTests, tests);
        atomicAdd(A.stats + kStatVotes, votes);
        if (threadIdx.x == 0) {
            A.counts[0] = nt;
            A.stats[kStatVisited0] = nt;
            A.stats[kStatSplit0] = carry_f;
        }
    }
    grid.sync();
    if (A.pts && *(volatile uint32_t*)(A.ctl + 3)) {        // every thread reads the same flag
        grid.sync();                                         // ... before it is re-armed
        if (gtid == 0) {
            A.ctl[3] = 0;
            A.fin[0] = 1;
            __threadfence_system();
        }
        return;
    }
    mid_pass<I, true>(A, 0, 0, A.ctl[1], warp, nwarps, lane, false);
    grid.sync();
    for (int l = 0; l < D; ++l) {
        const int cur = l & 1, nxt = cur ^ 1;
        const uint32_t F = A.ctl[4 * cur];
        if (F == 0) break;
        const uint32_t C = A.ctl[4 * cur + 1];
        const bool leaf = l + 1 == D;
        const uint32_t nk = 4 * F, ntiles = (F + blockDim.x - 1) / blockDim.x;   // a tile: one parent per thread
        // ---- S1: records, split flags, tile-local scans (thread = parent, its 4 children)
        if (threadIdx.x == 0) { s_acc[0] = 0; s_acc[1] = 0; }
        __syncthreads();
        for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const uint32_t r = tile * blockDim.x + threadIdx.x;
            uint4 v4 = make_uint4(0, 0, 0, 0);
            if (r < F) {
                v4 = *reinterpret_cast<const uint4*>(A.cv[cur] + 4 * r);
                if (A.record) {
                    const uint4 d0 = __ldg(A.fd[cur] + 2 * r);
                    const uint32_t t = d0.x & 0x7FFFFFFFu;
                    Record* rec = A.rec[l + 1] + 4ull * r;
                    rec[0] = {t, 2 * d0.y + 1, 2 * d0.z + 1, v4.x};      // NE
                    rec[1] = {t, 2 * d0.y, 2 * d0.z + 1, v4.y};          // NW
                    rec[2] = {t, 2 * d0.y, 2 * d0.z, v4.z};              // SW
                    rec[3] = {t, 2 * d0.y + 1, 2 * d0.z, v4.w};          // SE
                }
            }
            const uint32_t vv[4] = {v4.x, v4.y, v4.z, v4.w};
            Tri own{0, 0, 0}, loc[4];
            uint32_t my_v = 0, my_sv = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const bool split = r < F && (uint64_t)vv[q] > A.T;
                loc[q] = own;
                own.f += split ? 1u : 0u;
                own.s += split && !leaf ? vv[q] : 0u;
                own.c += split && !leaf ? (vv[q] + kChunk - 1) / kChunk : 0u;
                my_v += vv[q];
                my_sv += split && !leaf ? vv[q] : 0u;
            }
            Tri ex;
            const Tri tot = block_excl3(own, ex, s_w);
            if (r < F) {
                *reinterpret_cast<uint4*>(A.cursor + 4 * r) = make_uint4(ex.f + loc[0].f, ex.f + loc[1].f, ex.f + loc[2].f, ex.f + loc[3].f);
                *reinterpret_cast<uint4*>(A.loff + 4 * r) = make_uint4(ex.s + loc[0].s, ex.s + loc[1].s, ex.s + loc[2].s, ex.s + loc[3].s);
                *reinterpret_cast<uint4*>(A.lcoff + 4 * r) = make_uint4(ex.c + loc[0].c, ex.c + loc[1].c, ex.c + loc[2].c, ex.c + loc[3].c);
            }
            if (threadIdx.x == 0) { A.tiles[3 * tile] = tot.f; A.tiles[3 * tile + 1] = tot.s; A.tiles[3 * tile + 2] = tot.c; }
            const unsigned long long sv = __reduce_add_sync(0xFFFFFFFFu, my_v);   // 4 children < 2^28 (kMidMaxS)
            const unsigned long long ssv = __reduce_add_sync(0xFFFFFFFFu, my_sv);
            if (lane == 0) { atomicAdd(&s_acc[0], sv); atomicAdd(&s_acc[1], ssv); }
        }
        __syncthreads();
        if (threadIdx.x == 0 && (s_acc[0] || s_acc[1])) {
            atomicAdd(A.stats + kStatVotes, s_acc[0]);
            atomicAdd(A.stats + kStatTests, 4ull * s_acc[1]);
        }
        grid.sync();
        // ---- S2: tile prefixes (every block: one block scan over the tile totals, each thread holding
        // up to kMidMaxTiles / kMidThreads consecutive tiles), next frontier or leaves, child -> index
        {
            constexpr uint32_t kPer = (kMidMaxTiles + kMidThreads - 1) / kMidThreads;
            const uint32_t t0 = threadIdx.x * kPer;
            uint32_t tf[kPer], ts[kPer], tc[kPer];
            Tri own{0, 0, 0};
#pragma unroll
            for (uint32_t j = 0; j < kPer; ++j) {
                const bool ok = t0 + j < ntiles;
                tf[j] = ok ? A.tiles[3 * (t0 + j)] : 0u;
                ts[j] = ok ? A.tiles[3 * (t0 + j) + 1] : 0u;
                tc[j] = ok ? A.tiles[3 * (t0 + j) + 2] : 0u;
            }
#pragma unroll
            for (uint32_t j = 0; j < kPer; ++j) {
                if (t0 + j < ntiles) { s_pref[3 * (t0 + j)] = own.f; s_pref[3 * (t0 + j) + 1] = own.s; s_pref[3 * (t0 + j) + 2] = own.c; }
                own.f += tf[j]; own.s += ts[j]; own.c += tc[j];
            }
            Tri ex;
            const Tri tot = block_excl3(own, ex, s_w);
#pragma unroll
            for (uint32_t j = 0; j < kPer; ++j)
                if (t0 + j < ntiles) { s_pref[3 * (t0 + j)] += ex.f; s_pref[3 * (t0 + j) + 1] += ex.s; s_pref[3 * (t0 + j) + 2] += ex.c; }
            if (threadIdx.x == 0) { s_tot[0] = tot.f; s_tot[1] = tot.s; s_tot[2] = tot.c; }
            __syncthreads();
        }
        const uint32_t Fn = s_tot[0], Sn = s_tot[1], Cn = s_tot[2];
        for (uint32_t k = (uint32_t)gtid; k < nk; k += (uint32_t)gsize) {
            const uint32_t r = k >> 2, q = k & 3;
            const uint32_t tile = r / blockDim.x;
            const uint32_t v = A.cv[cur][k];
            const bool split = (uint64_t)v > A.T;
            if (!split) { A.cursor[k] = kNone; continue; }
            const uint32_t g = s_pref[3 * tile] + A.cursor[k];
            const uint4 d0 = __ldg(A.fd[cur] + 2 * r);
            const uint32_t t = d0.x & 0x7FFFFFFFu;
            const uint32_t ca = 2 * d0.y + quad_da((int)q), cc = 2 * d0.z + quad_dc((int)q);
            if (leaf) {
                A.leaves[g] = {t, ca, cc, v};
            } else {
                const uint32_t co = s_pref[3 * tile + 2] + A.lcoff[k];
                put_desc(A.fd[nxt], g, t, (d0.x >> 31) != 0, ca, cc, s_pref[3 * tile + 1] + A.loff[k], v, co);
                for (uint32_t q2 = 0, nc = (v + kChunk - 1) / kChunk; q2 < nc; ++q2) A.chunkmap[nxt][co + q2] = g;
                A.app[g] = 0;
                *reinterpret_cast<uint4*>(A.cv[nxt] + 4 * g) = make_uint4(0, 0, 0, 0);
            }
            A.cursor[k] = g;
        }
        if (gtid == 0) {
            A.counts[l + 1] = nk;
            A.stats[kStatVisited0 + l + 1] = nk;
            if (leaf) {
                A.counts[D + 1] = Fn;
                A.stats[kStatLeaves] = Fn;
            } else {
                A.stats[kStatSplit0 + l + 1] = Fn;
                A.ctl[4 * nxt] = Fn;
                A.ctl[4 * nxt + 1] = Cn;
                A.ctl[4 * nxt + 2] = Sn;
            }
        }
        grid.sync();
        if (leaf) break;
        // ---- W: append to the split children's lists, count their grandchildren
        if (Fn) mid_pass<I, false>(A, l, cur, C, warp, nwarps, lane, l + 2 < D);
        grid.sync();
    }
    // ---- results in the same launch: counts and statistics straight into the mapped host block (fin)
    if (A.fin && blockIdx.x == 0) {
        for (int i = threadIdx.x; i < D + 2; i += blockDim.x) A.fin[1 + i] = A.counts[i];
        unsigned long long* hs = reinterpret_cast<unsigned long long*>(A.fin + kFinishStatsWord);
        for (int i = threadIdx.x; i < kStatCount; i += blockDim.x) hs[i] = A.stats[i];
        if (threadIdx.x == 0) A.fin[0] = 0;
        __threadfence_system();
    }
}
}  // namespace

int mid_blocks_per_sm(bool int64) {
    int n = 0;
    if (int64) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_mid<int64_t>, kMidThreads, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_mid<int32_t>, kMidThreads, 0);
    return n > 0 ? n : 1;
}

cudaError_t launch_mid(const MidArgs& a, bool int64, int grid, cudaStream_t st) {
    void* args[] = {(void*)&a};
    return cudaLaunchCooperativeKernel(int64 ? (const void*)k_mid<int64_t> : (const void*)k_mid<int32_t>,
                                       dim3(grid), dim3(kMidThreads), args, 0, st);
}

}  // namespace hht

// Device kernels of the level-synchronous hierarchical Hough pass (sm_100a).
//
// Paper: Singh & Bhatia, arXiv 1007.0547. What each kernel computes, in the paper's
// terms, and the readings it rests on are in DESIGN.md §4; the oracle that checks it is oracle/
// (shares nothing with this file).
//
// Integer formulation: for an effective point (ex, ey) (BETA swaps,
// PAPER.md:67) and lattice corner (i, j) with m_i = -1 + 2i/2^D, b_j = -N + 3N*j/2^D,
//     G(i, j) = 2^D*(ey - ex*m_i - b_j) = 2^D*(ex + ey + N) - 2*i*ex - 3N*j,
// and the corner is below the line b = ey - ex*m (its getcode() bit is 1) iff G > 0.
// Because 0 <= ex < N < 1.5N, every region satisfies G_SW >= G_SE > G_NW >= G_NE, so its code is
// one of 0000, 0010, 0011, 0111, 1111 and "code != 0000 and != 1111" is exactly
// G_SW > 0 >= G_NE, i.e. 0 < G_SW <= s*(2ex + 3N) for a region of side s. In unsigned arithmetic
// that is the single compare (G_SW - 1) <u s*(2ex + 3N). The children of a region with SW value g
// have SW values g - {0, Pc} - {0, Qc} (Pc = ex*s, Qc = 3N*s/2): the 9 lattice points of the
// region (corners, edge midpoints, centre) decide the parent code and all four child codes.
#include <algorithm>
#include <cooperative_groups.h>
#include <cuda/atomic>

#include "hht_internal.h"

namespace hht {

namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;

template <typename I> struct Unsigned;
template <> struct Unsigned<int32_t> { using type = uint32_t; };
template <> struct Unsigned<int64_t> { using type = uint64_t; };

// 0 < v <= U  <=>  (v - 1) <u U  (v > -2^(bits-1) guaranteed by the width check).
template <typename I>
__device__ __forceinline__ bool crosses(I v_minus_1, I U) {
    using UI = typename Unsigned<I>::type;
    return (UI)v_minus_1 < (UI)U;
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
    uint32_t lo = __shfl_sync(kFull, (uint32_t)v, src), hi = __shfl_sync(kFull, (uint32_t)(v >> 32), src);
    return ((uint64_t)hi << 32) | lo;
}

// Warp sum of four byte counters packed in one word (each <= 255 per lane, sums < 2^16).
// Returns counter `which` (0..3) of the warp total; all lanes must call.
__device__ __forceinline__ void warp_sum_bytes(uint32_t acc, uint32_t& c02, uint32_t& c13) {
    c02 = __reduce_add_sync(kFull, acc & 0x00FF00FFu);
    c13 = __reduce_add_sync(kFull, (acc >> 8) & 0x00FF00FFu);
}
__device__ __forceinline__ uint32_t byte_counter(uint32_t c02, uint32_t c13, int which) {
    return (((which & 1) ? c13 : c02) >> (16 * (which >> 1))) & 0xFFFFu;
}

// quad index of (da, dc): NE(1,1)=0, NW(0,1)=1, SW(0,0)=2, SE(1,0)=3
__host__ __device__ constexpr int quad_of(int da, int dc) { return dc ? (da ? 0 : 1) : (da ? 3 : 2); }

}  // namespace

// ---------------------------------------------------------------------------------------------
// K0: stage and validate (SPEC.md:310 rejects out-of-range points before any
// traversal). Packs (x, y) into one word x << 16 | y; the BETA swap happens at use.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_stage(const int2* __restrict__ pts, uint64_t n, int N,
                                               uint32_t* __restrict__ packed, uint32_t* __restrict__ err) {
    uint32_t bad = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int2 p = __ldcs(pts + i);
        const bool ok = (unsigned)p.x < (unsigned)N && (unsigned)p.y < (unsigned)N;
        bad |= !ok;
        packed[i] = ok ? (((uint32_t)p.x << 16) | (uint32_t)p.y) : 0u;
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

cudaError_t launch_stage(const int32_t* pts, uint64_t n, int N, uint32_t* packed, uint32_t* err,
                         cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_stage<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const int2*>(pts), n, N, packed, err);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// K1/K4 fused: one pass over the candidate lists of the split regions at parent level l.
//
// One warp owns one chunk (<= 256 consecutive entries of ONE region's list; 8 per lane, loaded
// coalesced with streaming hints). Per entry it evaluates the region's 9-point lattice signs in
// the reduced form above and
//   MODE_COUNT  : counts votes of the 4 children (used at the root, PAPER.md steps 1-5 / 12);
//   MODE_WRITE  : appends the entry to the list of every SPLIT child it crosses (PAPER.md:100-103
//                 "if the line passes through the parent region then decide about the child
//                 regions") with warp-aggregated atomics, and counts the votes of the children of
//                 those split children ("count-ahead": the next level's votes are produced while
//                 the entry is in registers, so each list is read exactly once);
//   MODE_COUNT2 : MODE_WRITE without the append (the children are at level D-1: their lists would
//                 only be read to count the leaves, which this pass already does).
// Votes are warp ballots / per-lane byte counters reduced with __reduce_add_sync and added with one
// atomic per (warp chunk, region, quad): a segmented reduction whose segments are chunks.
// ---------------------------------------------------------------------------------------------
// Per-entry arithmetic of one chunk (8 entries per lane). Invalid lanes (past the chunk's end) get
// g - 1 = -1, which crosses nothing, so the body is branch-free.
//   cm  : 4 child bits per item (MODE_COUNT / MODE_WRITE), item it at bits [4it, 4it+4)
//   acc : MODE_COUNT: acc[0] byte q = votes of child q; else acc[q] byte q' = votes of grandchild
//         q' of child q (count-ahead over the 4x4 level-(l+2) cells (u, v), SW value
//         g - u*Pg - v*Qg; containment makes the child's own crossing implied).
// Count-ahead raster (MODE_WRITE / MODE_COUNT2): the 4x4 level-(l+2) cells under a parent of side
// s = 2^sh are rastered like the 16x16 leaf grid (see "Fixed-point raster state" at Raster16), on
// y' = floor((g - 1) / 2^(sh-2)): with Pg = 2ex s/4 and Qg = 3N s/4, floor((y - u Pg) / Qg) =
// floor((y' - 2ex u) / 3N) because u Pg is a multiple of 2^(sh-2), so the leaf raster's fixed point
// (Y ~ 2^24 (y' / 3N + B), decrement P from 2ex) applies unchanged; y' < 4 (2ex + 3N) keeps the
// floors f in [-5, 6] over the 5 column boundaries. Column u's crossed rows f_(u+1) .. f_u (clipped
// to 0..3) come as 4 byte counters from a table indexed by t = f_u + f_(u+1), one 4-byte copy per lane.
constexpr int kTab4TLo = -12;   // t in [-12, 14)
constexpr int kTab4 = 26;
__shared__ uint32_t s_tab4[(kTab4 + 2) * 64];     // entries 256 B apart (32 lane words + 128 B gap)

struct Tab4Place {
    uint32_t H, B;
};

__device__ __forceinline__ Tab4Place tab4_place() {
    const uint32_t S = (uint32_t)__cvta_generic_to_shared(s_tab4);
    const uint32_t H = S & 0xFFFF0000u;
    uint32_t twoB = ((S - H + 255u) >> 8) + (uint32_t)(-kTab4TLo);
    twoB += twoB & 1u;
    return {H, twoB >> 1};
}

// entry t, lane copy c at H + 256 (t + 2B) + 4 c
__device__ __forceinline__ void fill_tab4() {
    const Tab4Place pl = tab4_place();
    const uint32_t first = pl.H + 256u * (uint32_t)(kTab4TLo + 2 * (int)pl.B);
    for (int i = threadIdx.x; i < kTab4 * 32; i += blockDim.x) {
        const int t = kTab4TLo + (i >> 5);
        const int f = t >= 0 ? (t + 1) / 2 : -((-t) / 2), fn = t - f;
        uint32_t w = 0;
        for (int v = max(fn, 0); v <= min(f, 3); ++v) w |= 1u << (8 * v);
        asm volatile("st.shared.u32 [%0], %1;" :: "r"(first + 256u * (uint32_t)(i >> 5) + 4u * (uint32_t)(i & 31)), "r"(w) : "memory");
    }
}

struct CARaster {
    uint32_t lane_h, bias, fx_m, fx_mlo, fx_s;
    __device__ __forceinline__ void init(const PassArgs& A, int lane) {
        const Tab4Place pl = tab4_place();
        lane_h = pl.H | (2u * (uint32_t)lane);     // two boundaries add up to the lane's word 4 lane
        bias = (pl.B << 24) + 1u;
        fx_m = A.fx_m;
        fx_mlo = A.fx_mlo;
        fx_s = A.fx_s;
    }
};

template <typename I, int MODE, bool BETA>
__device__ __forceinline__ void chunk_math(const uint32_t (&p)[kItems], int cnt, int lane, I alpha, I beta_m1,
                                           int D, int sh, I Qc, I Qg, uint32_t one, uint32_t& cm,
                                           uint32_t (&acc)[4], const CARaster& CR) {
    uint32_t col[4] = {0, 0, 0, 0};                   // count-ahead: col[u] byte v = cells (u, v)
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const uint32_t w = p[it];
        const I ex = (I)(BETA ? (w & 0xFFFFu) : (w >> 16));
        const I ey = (I)(BETA ? (w >> 16) : (w & 0xFFFFu));
        I gm1 = ex * alpha + (ey << D) + beta_m1;            // G(SW corner) - 1
        if (MODE != MODE_WRITE_NC && lane + kWarp * it >= cnt) gm1 = (I)-1;
        const I Pc = ex << sh;                                // ex * s
        if (MODE == MODE_WRITE_NC) {
            // every entry of a region's own list crosses it, so y = G_SW - 1 lies in [0, 2 Uc) and
            // the NE child (y >= Uc) is crossed exactly when the SW child (y < Uc) is not (the
            // SW + NE identity); NW and SE keep their exact tests. Lanes past the chunk are masked
            // once per chunk below (the fused tail's push does the same).
            const I Uc = Pc + Qc;
            const uint32_t b = (crosses<I>(gm1, Uc) ? 4u : 1u) | (crosses<I>(gm1 - Qc, Uc) << 1) |
                               (crosses<I>(gm1 - Pc, Uc) << 3);
            cm |= b << (4 * it);
        }
        if (MODE == MODE_COUNT) {
            const I Uc = Pc + Qc;
            // child SW values: NE g-Pc-Qc, NW g-Qc, SW g, SE g-Pc
            const uint32_t bNE = crosses<I>(gm1 - Pc - Qc, Uc);
            const uint32_t bNW = crosses<I>(gm1 - Qc, Uc);
            const uint32_t bSW = crosses<I>(gm1, Uc);
            const uint32_t bSE = crosses<I>(gm1 - Pc, Uc);
            acc[0] += bNE | (bNW << 8) | (bSW << 16) | (bSE << 24);
        }
        if (MODE == MODE_WRITE || MODE == MODE_COUNT2) {
            // the 4x4 level-(l+2) cells as a 4-column raster (CARaster above); invalid lanes keep
            // f = -1 (all-zero entries)
            // (Raster16's 32-bit multiply-high form of this setup measured slower here: 73 registers
            // instead of 64, 3 blocks/SM, C5 write passes 39.6 -> 40.4 ms)
            const bool valid = gm1 >= 0;
            const uint32_t y0 = (uint32_t)(gm1 >> (sh - 2));
            uint32_t Y = valid ? (uint32_t)(((uint64_t)y0 * CR.fx_m) >> CR.fx_s) + CR.bias : CR.bias - (1u << 24) - 1u;
            const uint32_t P = valid ? (uint32_t)(((uint64_t)(2u * (uint32_t)ex) * CR.fx_mlo) >> CR.fx_s) : 0u;
            uint32_t X = __byte_perm(Y, CR.lane_h, 0x7634u);          // boundary 0 carries H
            uint32_t mc[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                Y -= P;
                const uint32_t xn = __byte_perm(Y, CR.lane_h, (u & 1) ? 0x7634u : 0x5534u);
                uint32_t addr;
                asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(addr) : "r"(X), "r"(one), "r"(xn));
                asm("ld.shared.u32 %0, [%1];" : "=r"(mc[u]) : "r"(addr));
                X = xn;
                col[u] += mc[u];
            }
            if (MODE == MODE_WRITE) {
                // child bits from the same cells: a line crosses a child iff it crosses one of the
                // child's 4 cells (the children tile it; SW + NE identity). Child (da, dc) = columns
                // 2da, 2da+1 x rows 2dc, 2dc+1. Bytes of x: NE, NW, SW, SE (each 0/1); the multiply
                // gathers byte k's bit to bit 28 + k.
                const uint32_t a = mc[0] | mc[1], b = mc[2] | mc[3];
                const uint32_t x = __byte_perm(a, b, 0x4026u) | __byte_perm(a, b, 0x5137u);
                const uint32_t nib = (x * 0x10204080u) >> 28;
                cm |= nib << (4 * it);
            }
        }
    }
    if (MODE == MODE_WRITE_NC) {
        const int nv = cnt - lane;                            // valid items of this lane: ceil(nv / 32)
        const int kv = nv <= 0 ? 0 : min((nv + kWarp - 1) / kWarp, kItems);
        cm &= kv >= kItems ? 0xFFFFFFFFu : ((1u << (4 * kv)) - 1u);
    }
    if (MODE == MODE_WRITE || MODE == MODE_COUNT2) {
        // acc[q] byte qq = cell (2 da_q + da_qq, 2 dc_q + dc_qq); quads NE(1,1) NW(0,1) SW(0,0) SE(1,0)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int da = quad_da(q), dc = quad_dc(q);
            acc[q] = __byte_perm(col[2 * da], col[2 * da + 1], dc ? 0x6237u : 0x4015u);
        }
    }
}

#ifndef HHT_DESC_NOPAD
#define HHT_DESC_NOPAD 1
#endif
// Chunk descriptor (32 B, one broadcast load per warp) and the chunk's entries. Lanes past `cnt`
// load nothing; a descriptor past the launch's chunk range reads as cnt = 0.
__device__ __forceinline__ ChunkDesc load_desc(const ChunkDesc* __restrict__ d, uint64_t ch, uint64_t c_hi) {
    ChunkDesc z;
    if (ch < c_hi) {
        const uint4* q = reinterpret_cast<const uint4*>(d + ch);
#if HHT_DESC_NOPAD
        // the unused pad word is not loaded: a vector load's dead destination register is reused by
        // the compiler right away, and that write then waits (write-after-write on the scoreboard)
        // for the load of a descriptor two chunks ahead (ncu, C5 last list pass: 27 % of all stall
        // samples on two such instructions)
        // (the flag word through a plain global load: ptxas merges adjacent non-coherent loads of the
        // same kind back into one 128-bit load)
        const uint4 u0 = __ldg(q);
        const uint2 e = __ldg(reinterpret_cast<const uint2*>(q + 1));
        uint32_t beta;
        asm("ld.global.u32 %0, [%1];" : "=r"(beta) : "l"(reinterpret_cast<const uint32_t*>(q + 1) + 2));
        z.r = u0.x; z.cnt = u0.y; z.a = u0.z; z.c = u0.w;
        z.e0 = ((uint64_t)e.y << 32) | e.x;
        z.beta = beta; z.pad = 0;
#else
        const uint4 u0 = __ldg(q), u1 = __ldg(q + 1);
        z.r = u0.x; z.cnt = u0.y; z.a = u0.z; z.c = u0.w;
        z.e0 = ((uint64_t)u1.y << 32) | u1.x;
        z.beta = u1.z; z.pad = 0;
#endif
    } else {
        z.r = 0; z.cnt = 0; z.a = 0; z.c = 0; z.e0 = 0; z.beta = 0; z.pad = 0;
    }
    return z;
}

__device__ __forceinline__ void load_items(uint32_t (&p)[kItems], const uint32_t* __restrict__ list, uint64_t base,
                                           const ChunkDesc& d, int lane) {
    const uint32_t* src = list + (d.e0 - base) + lane;       // one 64-bit address, immediate offsets
#pragma unroll
    for (int it = 0; it < kItems; ++it) p[it] = (lane + kWarp * it < (int)d.cnt) ? __ldcs(src + kWarp * it) : 0u;
}

// if (m != 0) { shared[sa] = v; sa += 4; }  -- predicated STS (the staging of the list compaction)
__device__ __forceinline__ void sts_if(uint32_t m, uint32_t& sa, uint32_t v) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p st.shared.u32 [%0], %2;\n\t@p add.u32 %0, %0, 4;\n\t}"
                 : "+r"(sa) : "r"(m), "r"(v) : "memory");
}

// Work loop of the pass and tail kernels: each warp walks chunks c_lo + warp0, + nwarps, ...; the
// next chunk's descriptor and entries are in flight while the current chunk is processed
// (PREF = true), or only the descriptor is (PREF = false, fewer registers).
struct NoAhead {
    __device__ __forceinline__ void operator()(const ChunkDesc&) const {}
};

// `ahead(dn)` is called with the next chunk's descriptor before the current chunk's body (and with
// the first chunk's before the loop): per-chunk loads that only depend on the descriptor (the
// list passes' child maps) are issued one chunk ahead there.
// L2PF: lane 0 also keeps the entry span of the chunk two ahead and hands it to the TMA unit as an
// L2 prefetch (cp.async.bulk.prefetch.L2: no registers or shared memory receive it), so the register
// loads of that chunk one iteration later hit L2.
__device__ __forceinline__ void span_of(const ChunkDesc* __restrict__ d, uint64_t ch, uint64_t c_hi, uint64_t& e0,
                                        uint32_t& cnt) {
    if (ch < c_hi) {
        const uint32_t* q = reinterpret_cast<const uint32_t*>(d + ch);
        cnt = __ldg(q + 1);
        const uint2 e = __ldg(reinterpret_cast<const uint2*>(q + 4));
        e0 = ((uint64_t)e.y << 32) | e.x;
    } else {
        cnt = 0;
        e0 = 0;
    }
}
__device__ __forceinline__ void l2_prefetch_span(const PassArgs& A, uint64_t e0, uint32_t cnt) {
    if (cnt == 0) return;
    const uint64_t e = e0 - A.list_base;
    const uint32_t off = (uint32_t)(e & 3u);
    const uint32_t bytes = ((off + cnt) * 4u + 15u) & ~15u;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(A.list + (e - off)), "r"(bytes) : "memory");
}

template <bool PREF, typename Body, typename Ahead = NoAhead, bool L2PF = false>
__device__ __forceinline__ void chunk_loop(const PassArgs& A, int lane, Body body, Ahead ahead = NoAhead{}) {
    const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t c_lo = A.chunk_bounds[0], c_hi = A.chunk_bounds[1];
    uint64_t ch = c_lo + warp0;
    ChunkDesc d = load_desc(A.chunks, ch, c_hi);
    ChunkDesc dn = load_desc(A.chunks, ch + nwarps, c_hi);
    uint32_t p[kItems];
    load_items(p, A.list, A.list_base, d, lane);
    ahead(d);
    uint64_t pf_e0 = 0;
    uint32_t pf_cnt = 0;
    if (L2PF && lane == 0) span_of(A.chunks, ch + 2 * nwarps, c_hi, pf_e0, pf_cnt);
    for (; ch < c_hi; ch += nwarps) {
        if (L2PF && lane == 0) {
            l2_prefetch_span(A, pf_e0, pf_cnt);          // chunk ch + 2 nwarps
            span_of(A.chunks, ch + 3 * nwarps, c_hi, pf_e0, pf_cnt);
        }
        if (PREF) {
            uint32_t pn[kItems];
            load_items(pn, A.list, A.list_base, dn, lane);
            const ChunkDesc dnn = load_desc(A.chunks, ch + 2 * nwarps, c_hi);
            ahead(dn);
            body(d, p);
#pragma unroll
            for (int it = 0; it < kItems; ++it) p[it] = pn[it];
            d = dn;
            dn = dnn;
        } else {
            ahead(dn);
            body(d, p);
            d = dn;
            dn = load_desc(A.chunks, ch + 2 * nwarps, c_hi);
            load_items(p, A.list, A.list_base, d, lane);
        }
    }
}

// TMA variant of the work loop (opts.prefetch 3, list passes): a per-warp ring of two shared-memory
// slots, each filled by one 1-D bulk copy (cp.async.bulk, one elected lane, completion counted on the
// slot's mbarrier) with the 16-byte-aligned span of a chunk's entries. While chunk k is processed
// from registers, the bulk copies of chunks k+1 and k+2 are in flight (2 KB per warp instead of the
// register prefetch's 1 KB), and no registers hold them.
constexpr uint32_t kTmaSlot = 1040;            // (3 + 256) words rounded up to 16 bytes
constexpr uint32_t kTmaWarpBytes = 2 * kTmaSlot + 16;   // two slots + two mbarriers

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    } while (!done);
}
// lane 0: bulk-copy the aligned span of chunk d's entries into slot `dst` (nothing for an empty chunk)
__device__ __forceinline__ void tma_chunk(const PassArgs& A, const ChunkDesc& d, uint32_t dst, uint32_t bar) {
    if (d.cnt == 0) return;
    const uint64_t e = d.e0 - A.list_base;
    const uint32_t off = (uint32_t)(e & 3u);
    const uint32_t bytes = ((off + d.cnt) * 4u + 15u) & ~15u;
    const uint32_t* src = A.list + (e - off);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

template <typename Body>
__device__ __forceinline__ void chunk_loop_tma(const PassArgs& A, int lane, uint32_t ring, Body body) {
    const uint64_t warp0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t c_lo = A.chunk_bounds[0], c_hi = A.chunk_bounds[1];
    const uint32_t bar0 = ring + 2 * kTmaSlot, bar1 = bar0 + 8;
    if (lane == 0) {
        mbar_init(bar0, 1);
        mbar_init(bar1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint64_t ch = c_lo + warp0;
    ChunkDesc d0 = load_desc(A.chunks, ch, c_hi);             // chunk k (slot k & 1)
    ChunkDesc d1 = load_desc(A.chunks, ch + nwarps, c_hi);    // chunk k + 1
    if (lane == 0) {
        tma_chunk(A, d0, ring, bar0);
        tma_chunk(A, d1, ring + kTmaSlot, bar1);
    }
    ChunkDesc d2 = load_desc(A.chunks, ch + 2 * nwarps, c_hi);
    uint32_t phase = 0;                                       // parity of the slot's current use
    for (uint32_t k = 0; ch < c_hi; ch += nwarps, ++k) {
        const uint32_t s = k & 1u;
        const uint32_t slot = ring + s * kTmaSlot, bar = s ? bar1 : bar0;
        uint32_t p[kItems];
        if (d0.cnt) {
            mbar_wait(bar, (phase >> s) & 1u);
            phase ^= 1u << s;
            const uint32_t off = (uint32_t)((d0.e0 - A.list_base) & 3u);
#pragma unroll
            for (int it = 0; it < kItems; ++it) {
                const uint32_t w = off + (uint32_t)lane + kWarp * it;
                uint32_t v = 0;
                if (lane + kWarp * it < (int)d0.cnt) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(slot + 4u * w));
                p[it] = v;
            }
        } else {
#pragma unroll
            for (int it = 0; it < kItems; ++it) p[it] = 0u;
        }
        __syncwarp();
        // the slot is free again: refill it with chunk k + 2 (generic reads before async writes)
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tma_chunk(A, d2, slot, bar);
        }
        const ChunkDesc d3 = load_desc(A.chunks, ch + 3 * nwarps, c_hi);
        body(d0, p);
        d0 = d1;
        d1 = d2;
        d2 = d3;
    }
}

// ---------------------------------------------------------------------------------------------
// FHT circumcircle variant ("calculates the perpendicular
// distance to the line from the center of the region and compares it with the radius of the
// circle circumscribing the region"). Same lists and passes, membership test replaced: with
// L(i, j) = G(i, j) (the line's signed lattice value) and a region of side s' with doubled centre
// (i2, j2), the line meets the circumcircle iff (L2)^2 <= 2 s'^2 (4ex^2 + 9N^2), L2 = 2 L(centre),
// exactly in integers (the oracle's form). A child (da, dc) of a parent of side s with SW value g
// has L2 = 2g - Pc(2da+1) - Qc(2dc+1) (Pc = ex s, Qc = 3N s/2); a grandchild (u, v) has
// L2 = 2g - Pg(2u+1) - Qg(2v+1) (Pg = ex s/2, Qg = 3N s/4). Circles are nested (a child's
// circumcircle lies inside its parent's), so a child's votes are again counted over the parent's
// list; but the SW+NE identity of the exact test does not hold, so all 16 grandchildren are
// counted and the dense tail is not used. int32 when 10 N 2^D < 2^31 (|L2| < 2^31, L2^2 < 2^62);
// int64 otherwise, with a 128-bit square.
// ---------------------------------------------------------------------------------------------
template <typename I>
__device__ __forceinline__ bool circle_in(I L2, uint64_t rhs) {
    if (sizeof(I) == 4) {
        const int64_t l = (int64_t)L2;
        return (uint64_t)(l * l) <= rhs;
    } else {
        const uint64_t a = (uint64_t)(L2 < 0 ? -L2 : L2);
        return __umul64hi(a, a) == 0 && a * a <= rhs;
    }
}

// Variant 2 (HHT_FHT_CIRCLE_MB, reading R22): the same circle measured in the (m, b) units of the
// parameter space, where a region of lattice side s' is a 2s'/2^D x 3N s'/2^D rectangle. The line
// b = ey - ex m lies at distance |F(centre)| / sqrt(1 + ex^2) from the centre and the circumradius
// is sqrt(w^2 + h^2) / 2; squared and scaled by 4^(D+1): L2^2 <= (1 + ex^2)(4 + 9N^2) s'^2 with
// the same L2 = 2 G(centre) = -2^(D+1) F(centre). Compared in 128-bit (the right side reaches
// 2^126 at the largest admitted N, D; the driver rejects larger).
__device__ __forceinline__ bool circle_in_mb(int64_t L2, unsigned __int128 rhs) {
    const uint64_t a = (uint64_t)(L2 < 0 ? -L2 : L2);
    return (unsigned __int128)a * a <= rhs;
}

template <typename I, int MODE, bool BETA, int VAR>
__device__ __forceinline__ void chunk_math_circle(const uint32_t (&p)[kItems], int cnt, int lane, I alpha, I beta_m1,
                                                  int D, int sh, I N, I Qc, I Qg, uint32_t& cm, uint32_t (&acc)[4]) {
    const uint64_t nn9 = 9ull * (uint64_t)N * (uint64_t)N;
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const uint32_t w = p[it];
        const I ex = (I)(BETA ? (w & 0xFFFFu) : (w >> 16));
        const I ey = (I)(BETA ? (w >> 16) : (w & 0xFFFFu));
        const bool valid = lane + kWarp * it < cnt;
        // invalid lanes: L2 odd (2g = 1, ex = 0) against rhs = 0 never passes
        const I twog = valid ? 2 * (ex * alpha + (ey << D) + beta_m1 + 1) : (I)1;
        const uint64_t K = valid ? 4ull * (uint64_t)ex * (uint64_t)ex + nn9 : 0ull;   // 4ex^2 + 9N^2
        // variant 2: (1 + ex^2)(4 + 9N^2) < 2^67 in 128 bits
        const unsigned __int128 K2 = valid ? (unsigned __int128)(1ull + (uint64_t)ex * (uint64_t)ex) * (4ull + nn9)
                                           : (unsigned __int128)0;
        const I Pc = ex << sh;
        if (MODE != MODE_COUNT2) {
            const uint64_t rc = VAR == 1 ? K << (2 * sh - 1) : 0ull;            // 2 (s/2)^2 K
            const unsigned __int128 rc2 = VAR == 2 ? K2 << (2 * sh - 2) : 0;     // (s/2)^2 K2
            uint32_t b = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const I L2 = twog - Pc * (I)(2 * quad_da(q) + 1) - Qc * (I)(2 * quad_dc(q) + 1);
                const bool in = VAR == 1 ? circle_in<I>(L2, rc) : circle_in_mb((int64_t)L2, rc2);
                b |= (in ? 1u : 0u) << (MODE == MODE_COUNT ? 8 * q : q);
            }
            if (MODE == MODE_COUNT) acc[0] += b;
            else cm |= b << (4 * it);
        }
        if (MODE != MODE_COUNT) {
            const uint64_t rg = VAR == 1 ? K << (2 * sh - 3) : 0ull;            // 2 (s/4)^2 K
            const unsigned __int128 rg2 = VAR == 2 ? K2 << (2 * sh - 4) : 0;     // (s/4)^2 K2
            const I Pg = Pc >> 1;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const I L2 = twog - Pg * (I)(2 * u + 1) - Qg * (I)(2 * v + 1);
                    const bool in = VAR == 1 ? circle_in<I>(L2, rg) : circle_in_mb((int64_t)L2, rg2);
                    if (in) acc[quad_of(u >> 1, v >> 1)] += 1u << (8 * quad_of(u & 1, v & 1));
                }
            }
        }
    }
}

// (No minimum resident blocks: the compiler's allocation gives the count-ahead pass 64 registers and
// the last list pass 57, 4 blocks/SM. Measured on C5: forcing 5 blocks/SM on the last pass (48
// registers, 40 B of spills) 44.4 vs 40.3 ms of list passes; an explicit minimum of 1 let the
// count-ahead pass grow to 115 registers, 2 blocks/SM, 50.4 ms.)
#ifndef HHT_PASS_L2PF
#define HHT_PASS_L2PF 0        // L2 bulk prefetch of the chunk two ahead: 1 in the last list pass, 2 in every writing pass
#endif
#ifndef HHT_PASS_MAP_AHEAD
#define HHT_PASS_MAP_AHEAD 0   // child maps one chunk ahead: 1 in the last list pass, 2 in every writing pass
#endif
template <typename I, int MODE, int PF, int CIRCLE>
__global__ void __launch_bounds__(256) k_pass(const PassArgs A) {
    constexpr bool PREF = PF == 1;
    constexpr bool kWrites = MODE == MODE_WRITE || MODE == MODE_WRITE_NC;
    __shared__ uint32_t s_stage[kWrites ? 8 * 4 * kChunk : 1];   // 4 KB per warp
    const int lane = threadIdx.x & 31;
    const int D = A.D;
    const int sh = D - A.level;                       // log2 of the parent side s (>= 1)
    const I N = (I)A.N;
    const I Qc = ((I)3 * N) << (sh - 1);              // 3N * s/2: child b-step
    const I Qg = (MODE == MODE_COUNT) ? (I)0 : (((I)3 * N) << (sh - 2));   // 3N * s/4 (sh >= 2)
    const uint32_t stage_sa = (uint32_t)__cvta_generic_to_shared(s_stage) + (threadIdx.x >> 5) * (4 * kChunk * 4);
    const uint32_t cell_q = ((uint32_t)lane * 11u) >> 5;          // lane L < 12: child q = L / 3
    const uint32_t cell_qq = (uint32_t)lane - 3u * cell_q + 1u;    // grandchild qq = 1 + L % 3
    CARaster CR{};
    if (!CIRCLE && (MODE == MODE_WRITE || MODE == MODE_COUNT2)) {
        fill_tab4();
        __syncthreads();
        CR.init(A, lane);
    }

    // lanes 0..3: next-frontier index and list offset of child `lane` (split children only), loaded
    // one chunk ahead (kMapAhead) or when the chunk is processed
    constexpr bool kMapAhead = !CIRCLE && PF != 2 && (MODE == MODE_WRITE_NC ? HHT_PASS_MAP_AHEAD >= 1
                                                                 : (MODE != MODE_COUNT && HHT_PASS_MAP_AHEAD >= 2));
    uint32_t cur_nf = kNone, nx_nf = kNone;
    uint64_t cur_off = 0, nx_off = 0;
    auto ahead = [&](const ChunkDesc& dn) {
        if (kMapAhead) {
            cur_nf = nx_nf;
            cur_off = nx_off;
            if (lane < 4 && dn.cnt != 0) {
                const uint64_t k = 4 * (uint64_t)(dn.r - A.nf_rbase) + lane;
                nx_nf = __ldg(A.nf + k);
                if (kWrites) nx_off = __ldg(A.nfoff + k);
            }
        }
    };

    auto body = [&](const ChunkDesc& d, const uint32_t (&p)[kItems]) {
        const int cnt = (int)d.cnt;
        const I i0 = (I)d.a << sh;
        const I j0 = (I)d.c << sh;
        const I alpha = ((I)1 << D) - 2 * i0;          // g = ex*alpha + (ey << D) + beta_c
        const I beta_m1 = (N << D) - (I)3 * N * j0 - 1;

        uint32_t my_nf = kNone;
        uint64_t my_off = 0;
        if (kMapAhead) {
            my_nf = cur_nf;
            my_off = cur_off;
        } else if (MODE != MODE_COUNT && lane < 4) {
            const uint64_t k = 4 * (uint64_t)(d.r - A.nf_rbase) + lane;
            my_nf = __ldg(A.nf + k);
            if (kWrites) my_off = __ldg(A.nfoff + k);
        }

        uint32_t cm = 0;
        uint32_t acc[4] = {0, 0, 0, 0};
        if (CIRCLE) {
            if (d.beta) chunk_math_circle<I, MODE, true, CIRCLE>(p, cnt, lane, alpha, beta_m1, D, sh, N, Qc, Qg, cm, acc);
            else chunk_math_circle<I, MODE, false, CIRCLE>(p, cnt, lane, alpha, beta_m1, D, sh, N, Qc, Qg, cm, acc);
        } else {
            if (d.beta) chunk_math<I, MODE, true>(p, cnt, lane, alpha, beta_m1, D, sh, Qc, Qg, A.one, cm, acc, CR);
            else chunk_math<I, MODE, false>(p, cnt, lane, alpha, beta_m1, D, sh, Qc, Qg, A.one, cm, acc, CR);
        }

        if (MODE == MODE_COUNT) {
            uint32_t c02, c13;
            warp_sum_bytes(acc[0], c02, c13);
            if (lane < 4) {
                const uint32_t v = byte_counter(c02, c13, lane);
                if (v) atomicAdd(A.votes + 4 * (uint64_t)(d.r - A.nf_rbase) + lane, v);
            }
            return;
        }

        if (my_nf != kNone && (my_nf < A.q0 || my_nf >= A.q1)) my_nf = kNone;

        if (MODE == MODE_WRITE_NC) {
            // no count-ahead: the next level's votes come from the fused tail's leaf grids
        } else if (CIRCLE) {
            // all 16 grandchild cells (no derivation for circles): cell L = 4q + qq at field L & 1
            // of word L >> 1, one warp sum per word; lane L < 16 adds cell L
            uint32_t sw = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t lo = (acc[q] & 0xFFu) | ((acc[q] << 8) & 0xFF0000u);
                const uint32_t hi = ((acc[q] >> 16) & 0xFFu) | ((acc[q] >> 8) & 0xFF0000u);
                const uint32_t slo = __reduce_add_sync(kFull, lo), shi = __reduce_add_sync(kFull, hi);
                if ((lane >> 2) == q) sw = (lane & 2) ? shi : slo;
            }
            const uint32_t v = (sw >> (16 * (lane & 1))) & 0xFFFFu;
            const uint32_t nf_l = __shfl_sync(kFull, my_nf, (lane >> 2) & 3);
            if (lane < 16 && nf_l != kNone && v) atomicAdd(A.votes + 4 * (uint64_t)(nf_l - A.q0) + (lane & 3), v);
        } else
        // Count-ahead votes: the 12 derived-free cells (child q, grandchild qq = NW, SW, SE) in
        // 16-bit fields of 6 words (cell L = 3q + qq - 1 at field L & 1 of word L >> 1), one warp
        // sum per word; lane L < 12 then adds cell L to its split child's vote counter.
        {
            const uint32_t w0 = ((acc[0] >> 8) & 0xFFu) | (acc[0] & 0xFF0000u);
            const uint32_t w1 = (acc[0] >> 24) | ((acc[1] << 8) & 0xFF0000u);
            const uint32_t w2 = ((acc[1] >> 16) & 0xFFu) | ((acc[1] >> 8) & 0xFF0000u);
            const uint32_t w3 = ((acc[2] >> 8) & 0xFFu) | (acc[2] & 0xFF0000u);
            const uint32_t w4 = (acc[2] >> 24) | ((acc[3] << 8) & 0xFF0000u);
            const uint32_t w5 = ((acc[3] >> 16) & 0xFFu) | ((acc[3] >> 8) & 0xFF0000u);
            const uint32_t s0 = __reduce_add_sync(kFull, w0), s1 = __reduce_add_sync(kFull, w1);
            const uint32_t s2 = __reduce_add_sync(kFull, w2), s3 = __reduce_add_sync(kFull, w3);
            const uint32_t s4 = __reduce_add_sync(kFull, w4), s5 = __reduce_add_sync(kFull, w5);
            const uint32_t t0 = (lane & 2) ? s1 : s0, t1 = (lane & 2) ? s3 : s2, t2 = (lane & 2) ? s5 : s4;
            const uint32_t sw = (lane & 8) ? t2 : ((lane & 4) ? t1 : t0);      // word lane >> 1 (lane < 12)
            const uint32_t v = (sw >> (16 * (lane & 1))) & 0xFFFFu;
            const uint32_t nf_l = __shfl_sync(kFull, my_nf, cell_q);
            if (lane < 12 && nf_l != kNone && v) atomicAdd(A.votes + 4 * (uint64_t)(nf_l - A.q0) + cell_qq, v);
        }

        if (kWrites) {
            // Child list compaction (warp-private, order within a child list is irrelevant to the
            // counts): per-lane per-child counts -> one packed warp scan -> predicated stores into a
            // per-child shared-memory staging area -> one atomic per (chunk, split child) reserves a
            // run -> coalesced copy-out.
            uint32_t splitm = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) splitm |= (__shfl_sync(kFull, my_nf, q) != kNone ? 1u : 0u) << q;
            cm &= splitm * 0x11111111u;
            const uint32_t c0 = __popc(cm & 0x11111111u), c1 = __popc(cm & 0x22222222u);
            const uint32_t c2 = __popc(cm & 0x44444444u), c3 = __popc(cm & 0x88888888u);
            // inclusive scan of the 4 counts in byte fields: a lane's inclusive sum <= 31*8 except
            // lane 31's, whose wrap is undone exactly by the modular subtraction below
            const uint32_t own = c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
            uint32_t inc = own;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                uint32_t t;
                asm volatile("{\n\t.reg .pred p;\n\tshfl.sync.up.b32 %0|p, %1, %2, 0, 0xffffffff;\n\t@!p mov.b32 %0, 0;\n\t}"
                             : "=r"(t) : "r"(inc), "r"(dd));
                inc += t;
            }
            const uint32_t exc = inc - own;
            const uint32_t t02 = __reduce_add_sync(kFull, c0 | (c2 << 16));
            const uint32_t t13 = __reduce_add_sync(kFull, c1 | (c3 << 16));
            const uint32_t tq[4] = {t02 & 0xFFFFu, t13 & 0xFFFFu, t02 >> 16, t13 >> 16};
            // reserve the runs first: the staging stores below cover the atomics' round trip
            uint32_t my_base = 0;
            if (lane < 4) {
                const uint32_t t = lane == 0 ? tq[0] : lane == 1 ? tq[1] : lane == 2 ? tq[2] : tq[3];
                if (t) my_base = atomicAdd(A.c_cursor + (my_nf - A.q0), t);
            }
            uint32_t sa[4] = {stage_sa + 4 * (exc & 0xFFu), stage_sa + 4 * (kChunk + ((exc >> 8) & 0xFFu)),
                              stage_sa + 4 * (2 * kChunk + ((exc >> 16) & 0xFFu)),
                              stage_sa + 4 * (3 * kChunk + (exc >> 24))};
#pragma unroll
            for (int it = 0; it < kItems; ++it) {
#pragma unroll
                for (int q = 0; q < 4; ++q) sts_if(cm & (1u << (4 * it + q)), sa[q], p[it]);
            }
            const uint64_t my_dst = my_off - A.c_list_base + my_base;
            __syncwarp();
            const uint32_t* stage = s_stage + (threadIdx.x >> 5) * (4 * kChunk);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t n = tq[q];
                if (n == 0) continue;                       // warp-uniform
                uint32_t* dst = A.c_list + shfl_u64(my_dst, q) + lane;     // immediate offsets below
                const uint32_t* src = stage + q * kChunk + lane;
#pragma unroll
                for (int it = 0; it < kItems; ++it) {
                    if ((uint32_t)(kWarp * it) >= n) break;                 // warp-uniform
                    if ((uint32_t)(lane + kWarp * it) < n) dst[kWarp * it] = src[kWarp * it];
                }
            }
            __syncwarp();
        }
    };
    if constexpr (PF == 2) {
        extern __shared__ uint4 s_tma_ring[];
        chunk_loop_tma(A, lane, (uint32_t)__cvta_generic_to_shared(s_tma_ring) + (threadIdx.x >> 5) * kTmaWarpBytes, body);
    } else {
        constexpr bool kL2pf = !CIRCLE && (MODE == MODE_WRITE_NC ? HHT_PASS_L2PF >= 1
                                                              : (MODE != MODE_COUNT && HHT_PASS_L2PF >= 2));
        if constexpr (kMapAhead) chunk_loop<PREF, decltype(body), decltype(ahead), kL2pf>(A, lane, body, ahead);
        else chunk_loop<PREF, decltype(body), NoAhead, kL2pf>(A, lane, body);
    }
}

// ---------------------------------------------------------------------------------------------
// Dense raster tail: one pass over the lists of the split regions R at level L = D-3 counts the
// votes of every level-D region inside R (an 8x8 grid); the visited level-(D-1) and level-D
// regions' votes are then gathered from the grid. A region's votes are the number of lines
// crossing it, and R's list holds every line that crosses anything inside R (containment), so the
// grid counts are exactly the paper's votes. Level D-2 lists are never materialised.
//
// Level D-1 from level D: with G_SW >= G_centre >= G_NE for every region, a line crosses region C
// iff it crosses exactly one of C's SW child (G_SW > 0 >= G_centre) and NE child
// (G_centre > 0 >= G_NE), so votes(C) = votes(SW child) + votes(NE child).
//
// Raster of one line over the 8x8 leaf grid of R (cell side = 1 lattice step): with
// y_w = G(i0+w, j0) - 1 (w = 0..8, y_(w+1) = y_w - 2ex) and k_w = #{v in 0..8 : 3N*v <= y_w},
// cell (u, v) is crossed iff v < k_u and v >= k_(u+1) - 1: the rows of column u run from
// k_(u+1)-1 to min(k_u, 8)-1. Since 2ex < 3N, k drops by at most 1 per column (drop <=> y_(u+1) <
// (k_u - 1)*3N), so the column's crossed-row byte mask depends only on (k_u, drop) and comes from a
// 36-entry shared-memory table (k in -8..9: a line below the grid keeps "dropping" harmlessly into
// all-zero entries). Per column: one subtract, one compare, one 8-byte table load, two adds.
// ---------------------------------------------------------------------------------------------
constexpr int kTab8 = 36;   // (k + 8) * 2 + drop, k in -8..9

__device__ __forceinline__ uint2 tab8_entry(int t) {
    const int k = t / 2 - 8, d = t & 1;
    uint32_t lo = 0, hi = 0;
    if (k >= 1) {
        const int vhi = min(k, 8) - 1, vlo = max(k - d - 1, 0);
        for (int v = vlo; v <= vhi; ++v) {
            if (v < 4) lo |= 1u << (8 * v);
            else hi |= 1u << (8 * (v - 4));
        }
    }
    return make_uint2(lo, hi);
}

template <typename I, bool BETA>
__device__ __forceinline__ void tail_math(const uint32_t (&p)[kItems], int cnt, int lane, I alpha, I beta_m1,
                                          int D, I N3, const uint2* __restrict__ tab, uint32_t (&a8)[16]) {
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const uint32_t w = p[it];
        const I ex = (I)(BETA ? (w & 0xFFFFu) : (w >> 16));
        const I ey = (I)(BETA ? (w >> 16) : (w & 0xFFFFu));
        I y = ex * alpha + (ey << D) + beta_m1;            // G(SW corner of R) - 1
        if (lane + kWarp * it >= cnt) y = (I)-1;            // crosses nothing
        const I P8 = 2 * ex;
        // f = min(floor(y / 3N), 8) for y >= 0 (branch-free binary search); k0 = f + 1 (0 if y < 0)
        I f = (y >= (I)4 * N3) ? (I)4 : (I)0;
        f += (y >= (f + 2) * N3) ? (I)2 : (I)0;
        f += (y >= (f + 1) * N3) ? (I)1 : (I)0;
        f = (y >= (I)8 * N3) ? (I)8 : f;
        const bool below = y < 0;
        I Kq = below ? -N3 : f * N3;                         // (k - 1) * 3N: drop threshold
        int kk = below ? 16 : 2 * (int)f + 18;               // table index of (k, 0): 2 * (k + 8)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            y -= P8;
            const bool drop = y < Kq;
            const uint2 m = tab[16 * (kk + (drop ? 1 : 0))];
            a8[2 * u] += m.x;
            a8[2 * u + 1] += m.y;
            if (drop) {
                kk -= 2;
                Kq -= N3;
            }
        }
    }
}

// Table replicated 16x (an LDS.64 serves 16 lanes per wavefront): lane l reads copy (l & 15).
template <typename I>
__global__ void __launch_bounds__(256) k_tail(const PassArgs A) {
    __shared__ uint2 s_tab[kTab8 * 16];
    for (int t = threadIdx.x; t < kTab8 * 16; t += blockDim.x) s_tab[t] = tab8_entry(t >> 4);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int D = A.D;
    const int sh = D - A.level;                       // == 3
    const I N = (I)A.N;
    const I N3 = (I)3 * N;

    chunk_loop<false>(A, lane, [&](const ChunkDesc& d, const uint32_t (&p)[kItems]) {
        const int cnt = (int)d.cnt;
        const I i0 = (I)d.a << sh;
        const I j0 = (I)d.c << sh;
        const I alpha = ((I)1 << D) - 2 * i0;
        const I beta_m1 = (N << D) - N3 * j0 - 1;
        uint32_t a8[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) a8[i] = 0;
        if (d.beta) tail_math<I, true>(p, cnt, lane, alpha, beta_m1, D, N3, s_tab + (lane & 15), a8);
        else tail_math<I, false>(p, cnt, lane, alpha, beta_m1, D, N3, s_tab + (lane & 15), a8);

        // grid[(r - nf_rbase) * 64 + 8u + v]: a8[2u] byte b = row b, a8[2u+1] byte b = row 4+b
        uint32_t* dst = A.votes + (uint64_t)(d.r - A.nf_rbase) * kTailCells;
#pragma unroll
        for (int wi = 0; wi < 16; ++wi) {
            uint32_t c02, c13;
            warp_sum_bytes(a8[wi], c02, c13);
            if (lane < 4) {
                const uint32_t v = byte_counter(c02, c13, lane);
                if (v) atomicAdd(dst + 8 * (wi >> 1) + 4 * (wi & 1) + lane, v);
            }
        }
    });
}

// ---------------------------------------------------------------------------------------------
// 16x16 dense tail (level L = D-4): the same raster over a 16x16 leaf grid. Every level below L+1
// then comes from the leaf grid: a line crosses a region iff it crosses exactly one of the region's
// diagonal (SW..NE) leaves (the SW+NE identity applied recursively), so
// votes(region of side 2^j leaves) = sum of its 2^j diagonal leaf counts.
// The 64 per-lane counter words do not fit in registers, so the grid is processed in 4 column
// blocks of 4 columns; each line's raster state (Y, P, X below) is carried across blocks, and
// each block's 8 nibble counter words are reduced across the warp with a butterfly reduce-scatter
// (12 shuffles) that leaves every lane with the warp totals of 2 cells.
// ---------------------------------------------------------------------------------------------
// Fixed-point raster state. For a line of the batch, y_u = G(i0 + u, j0) - 1 at lattice column u of
// the leaf grid and f_u = floor(y_u / 3N): the line is above lattice corner (u, v) (G > 0) iff
// v <= f_u, so it crosses cell (u, v) (G_SW > 0 >= G_NE) iff f_(u+1) <= v <= f_u, rows clipped to
// 0..15 (2ex < 3N, so f drops by 0 or 1 per column). The raster carries Y_u ~ 2^24 (y_u / 3N + B)
// in 32 bits, B a per-block bias: its top byte is f_u + B. One PRMT per column boundary turns Y_u
// into X_u = (f_u + B) << 8 | 4 lane, plus (at even boundaries) the table's 64 KB-aligned base H,
// and the table entry of column u (t = f_u + f_(u+1) = 2 f_u - drop, lane copy) sits at
// X_u + X_(u+1) = H + 256 (t + 2B) + 8 lane: a column step is Y -= P, PRMT, one 2-input add (an
// integer multiply-add by a runtime 1, FMA pipe), LDS.64.
// Exactness: every line of a batch crosses the 16x16 region, so 0 <= y_0 < 16 (2ex +
// 3N) < 32 * 3N <= 2^fx_s. Y_0 = floor(y_0 fx_m / 2^fx_s) + 1 with fx_m = ceil(2^(24+fx_s) / 3N)
// exceeds the exact value 2^24 y_0 / 3N by (0, 2); P = floor(2ex fx_mlo / 2^fx_s) with fx_mlo =
// floor(2^(24+fx_s) / 3N) falls below 2^24 2ex / 3N by [0, 2). So Y_u - 2^24 y_u / 3N lies in
// (0, 2 + 2u) subset (0, 34) for u <= 16, while a non-multiple of 3N sits at least 2^24 / 3N > 34
// units (3N < 493447) from the next multiple: floor(Y_u / 2^24) - B = f_u exactly. f_u stays in
// [-16, 26] (f_0 <= 26, one drop per column) and B in [17, 145], so the top byte never wraps.
constexpr int kTab16TLo = -34;  // table entries t = f_u + f_(u+1) in [-34, 56)
constexpr int kTab16 = 90;
constexpr int kTab16Slots = (kTab16 + 2) * 32;   // + 2 entries of slack for the placement below

// Column mask of the 16x16 tail as 4-bit counters, one table copy per lane. Logical row
// v = 8h + 2b + par (h: word, b: byte, par: nibble within the byte) is stored at word h ^ L4, byte
// b ^ L0, nibble par ^ L3, where Lx is bit x of the lane that owns the copy: the three lane-bit
// swaps are exactly the register swaps the butterfly reduce-scatter in Raster16 would otherwise do
// with selects (levels xor 16, xor 8 and the final xor 1). A lane adds at most 7 per cell per column
// block, so nibbles do not overflow; they are widened to bytes during the reduction.
__device__ __forceinline__ uint2 tab16_entry(int t, int lane) {
    const int f = t >= 0 ? (t + 1) / 2 : -((-t) / 2);  // f_u = ceil(t / 2)
    const int fn = t - f;                              // f_(u+1)
    uint32_t w[2] = {0, 0};
    {
        const int vhi = min(f, 15), vlo = max(fn, 0);  // crossed rows f_(u+1) .. f_u
        for (int v = vlo; v <= vhi; ++v) {
            const int hp = (v >> 3) ^ ((lane >> 4) & 1);
            const int bp = ((v >> 1) & 3) ^ (lane & 1);
            const int np = (v & 1) ^ ((lane >> 3) & 1);
            w[hp] |= 1u << (4 * (2 * bp + np));
        }
    }
    return make_uint2(w[0], w[1]);
}

// The raster's table (static shared memory of the kernels that raster) and its placement: with S
// its shared address, H = S rounded down to 64 KB and 2B the smallest even number >= ceil((S - H) /
// 256) - kTab16TLo, entry t of lane copy c lives at H + 256 (t + 2B) + 8 c, inside the array
// (0 <= H + 256 (kTab16TLo + 2B) - S < 512).
__shared__ uint2 s_tab16[kTab16Slots];

struct Tab16Place {
    uint32_t H, B;
};

__device__ __forceinline__ Tab16Place tab16_place() {
    const uint32_t S = (uint32_t)__cvta_generic_to_shared(s_tab16);
    const uint32_t H = S & 0xFFFF0000u;
    uint32_t twoB = ((S - H + 255u) >> 8) + (uint32_t)(-kTab16TLo);
    twoB += twoB & 1u;
    return {H, twoB >> 1};
}

__device__ __forceinline__ void fill_tab16() {
    const Tab16Place pl = tab16_place();
    const uint32_t first = pl.H + 256u * (uint32_t)(kTab16TLo + 2 * (int)pl.B);
    for (int i = threadIdx.x; i < kTab16 * 32; i += blockDim.x) {
        const uint2 e = tab16_entry(kTab16TLo + (i >> 5), i & 31);
        asm volatile("st.shared.v2.u32 [%0], {%1, %2};" :: "r"(first + 8u * (uint32_t)i), "r"(e.x), "r"(e.y) : "memory");
    }
}

// The 16x16 raster of one batch of <= 32 ITEMS lines over the leaf grid of one level-(D-4) region
// (a, c), accumulated into `dst` (256 u32 counters, [16 * column + row]) with one atomic per
// (lane, cell pair) per column block. Shared by the dense tail (batches = chunks of the region's
// list) and the fused tail (batches = full shared-memory stacks of a child of a level-(D-5) region).
#ifndef HHT_RASTER_ATOMIC_NOZ
#define HHT_RASTER_ATOMIC_NOZ 1     // 1: the two cell atomics per lane unconditionally (0: skip zero cells; slower)
#endif
#ifndef HHT_RASTER_VALID_BRANCH
#define HHT_RASTER_VALID_BRANCH 1   // 1: partial-batch lanes fixed up in a warp-uniform branch (0: per line)
#endif
#ifndef HHT_RASTER_SETUP_FMA
#define HHT_RASTER_SETUP_FMA 0      // 1: entry unpacking on the FMA pipe (multiply-high), not PRMT
#endif
#ifndef HHT_RASTER_XRECOMP
#define HHT_RASTER_XRECOMP 0      // 1: X of a column block's first boundary recomputed from Y (not carried)
#endif
template <typename I>
struct Raster16 {
    uint32_t lane_h, bias, red_u, red_row, fx_m, fx_mlo, fx_s, one;
    int D;
    I N, N3;

    __device__ __forceinline__ void init(const PassArgs& A, int lane) {
        const Tab16Place pl = tab16_place();
        lane_h = pl.H | (4u * (uint32_t)lane);       // byte 0: half the lane's copy offset; bytes 2-3: H
        bias = (pl.B << 24) + 1u;                    // Y_0 = floor(...) + 1 + B 2^24
        // cells this lane holds after the reduce-scatter: column 4b + u, u = L1 + 2 L2; rows
        // 8 L4 + 2 L0 + L3 (+ 4)
        red_u = ((lane >> 1) & 1) + 2 * ((lane >> 2) & 1);
        red_row = 8 * ((lane >> 4) & 1) + 2 * (lane & 1) + ((lane >> 3) & 1);
        fx_m = A.fx_m;
        fx_mlo = A.fx_mlo;
        fx_s = A.fx_s;
        one = A.one;
        D = A.D;
        N = (I)A.N;
        N3 = (I)3 * N;
    }

    // X_j of column boundary j: (f_j + B) << 8 | 4 lane, plus H at even j (exactly one of two
    // neighbouring boundaries carries the table base)
    __device__ __forceinline__ uint32_t boundary(uint32_t Yj, int j) const {
        return __byte_perm(Yj, lane_h, (j & 1) ? 0x5534u : 0x7634u);
    }

    // ITEMS lines per lane (a batch of <= 32 ITEMS). ITEMS <= 7 keeps every per-lane cell count
    // <= 7, so the first reduce-scatter level can add the 4-bit counters of two lanes before they
    // are widened to bytes (sums <= 14): half the widening work of that level. Larger batches
    // (<= 15 lines: 4-bit counts) exchange the raw nibble words and widen both before adding, so
    // that level still takes one shuffle per column.
    template <int ITEMS>
    __device__ __forceinline__ void run(const uint32_t (&p)[ITEMS], int cnt, uint32_t ra, uint32_t rc, uint32_t beta,
                                        uint32_t* dst, int lane) const {
        static_assert(ITEMS <= 15, "per-lane 4-bit cell counters hold at most 15 lines");
        const I i0 = (I)ra << 4;
        const I j0 = (I)rc << 4;
        const I alpha = ((I)1 << D) - 2 * i0;
        const I beta_m1 = (N << D) - N3 * j0 - 1;
        // byte selectors: ex = low half-word of the packed entry for BETA (x <-> y), high for ALPHA
        const uint32_t sel_ex = beta ? 0x4410u : 0x4432u, sel_ey = beta ? 0x4432u : 0x4410u;
        // y0 2^k (k = 32 - fx_s) in 32-bit modular arithmetic: exact, since 0 <= y0 < 2^fx_s for
        // every line of the batch, and then floor(y0 fx_m / 2^fx_s) = mulhi(y0 2^k, fx_m) (one
        // multiply-high with the bias as its addend); P likewise from 2ex 2^k = ex 2^(k+1)
        const uint32_t k = 32u - fx_s;
        const uint32_t alpha_s = (uint32_t)alpha << k;
        const uint32_t ey_s = ((uint32_t)D + k < 32u) ? (1u << ((uint32_t)D + k)) : 0u;
        const uint32_t beta_s = (uint32_t)beta_m1 << k;
        const uint32_t ex_s = 1u << (k + 1);

        // per-line state carried across the 4 column blocks: Y (fixed point, see above), its
        // per-column decrement P, and X of the previous column boundary
#if HHT_RASTER_XRECOMP
        uint32_t Y[ITEMS], P[ITEMS];                          // X recomputed at each block start
#else
        uint32_t Y[ITEMS], P[ITEMS], X[ITEMS];
#endif
#if HHT_RASTER_SETUP_FMA
        // unpack on the FMA pipe: hi = w >> 16 (multiply-high by an opaque 2^16), lo = w - hi 2^16,
        // with the half's coefficients chosen once per batch
        const uint32_t c_hi = beta ? ey_s : alpha_s, c_lo = beta ? alpha_s : ey_s;
        const uint32_t e_hi = beta ? 0u : ex_s, e_lo = beta ? ex_s : 0u;
        const uint32_t c16 = one << 16, m16 = 0u - c16;
#endif
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) {
            const uint32_t w = p[it];
#if HHT_RASTER_SETUP_FMA
            uint32_t hi, lo, y0s, pex;
            asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(w), "r"(c16));
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(lo) : "r"(hi), "r"(m16), "r"(w));
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(y0s) : "r"(hi), "r"(c_hi), "r"(beta_s));
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(y0s) : "r"(lo), "r"(c_lo), "r"(y0s));
            asm("mul.lo.u32 %0, %1, %2;" : "=r"(pex) : "r"(hi), "r"(e_hi));
            asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(pex) : "r"(lo), "r"(e_lo), "r"(pex));
#else
            const uint32_t ex = __byte_perm(w, 0, sel_ex);
            const uint32_t ey = __byte_perm(w, 0, sel_ey);
            const uint32_t y0s = ex * alpha_s + ey * ey_s + beta_s;         // (G(SW corner) - 1) 2^k
            const uint32_t pex = ex * ex_s;
#endif
            uint32_t yv, pv;
            asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(yv) : "r"(y0s), "r"(fx_m), "r"(bias));
            asm("mul.hi.u32 %0, %1, %2;" : "=r"(pv) : "r"(pex), "r"(fx_mlo));
#if HHT_RASTER_VALID_BRANCH
            Y[it] = yv;
            P[it] = pv;
#else
            const bool valid = lane + kWarp * it < cnt;
            // lanes past the batch: f = -1 in every column (all-zero entries)
            Y[it] = valid ? yv : bias - (1u << 24) - 1u;
            P[it] = valid ? pv : 0u;
#if !HHT_RASTER_XRECOMP
            X[it] = boundary(Y[it], 0);
#endif
#endif
        }
#if HHT_RASTER_VALID_BRANCH
        // lanes past a partial batch: f = -1 in every column (all-zero entries); full batches (the
        // common case) skip this warp-uniform block
        if (__builtin_expect(cnt < kWarp * ITEMS, 0)) {
#pragma unroll
            for (int it = 0; it < ITEMS; ++it) {
                if (lane + kWarp * it >= cnt) {
                    Y[it] = bias - (1u << 24) - 1u;
                    P[it] = 0u;
                }
            }
        }
#if !HHT_RASTER_XRECOMP
#pragma unroll
        for (int it = 0; it < ITEMS; ++it) X[it] = boundary(Y[it], 0);
#endif
#endif
#pragma unroll   // a rolled column-block loop (half the code, 44 B of spills) measured 151.7 vs 120.9 ms
        for (int b = 0; b < 4; ++b) {
            uint32_t acc[8];                                  // [2 * column-in-block + row half], nibbles
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = 0;
#pragma unroll
            for (int it = 0; it < ITEMS; ++it) {
#if HHT_RASTER_XRECOMP
                uint32_t Xc = boundary(Y[it], 0);                 // boundary 4b (even: carries H)
#else
                uint32_t& Xc = X[it];
#endif
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    Y[it] -= P[it];
                    const uint32_t xn = boundary(Y[it], 1 + u);   // boundary 4b + u + 1 (4b is even)
                    uint32_t addr, mx, my;
                    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(addr) : "r"(Xc), "r"(one), "r"(xn));
                    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(mx), "=r"(my) : "r"(addr));
                    Xc = xn;
                    acc[2 * u + 0] += mx;
                    acc[2 * u + 1] += my;
                }
            }
            // butterfly reduce-scatter over the lanes: xor 16 pairs the two physical words of a
            // column, xor 8 the two nibble parities, xor 4 and xor 2 the columns (selects), xor 1 the
            // byte pairs (0,2) / (1,3) split into 16-bit fields (sums <= 256). The per-lane table
            // layout makes "keep the first, send the second" correct for the select-free levels.
            uint32_t e1[4], o1[4];
            if (ITEMS <= 7) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {                 // xor 16 on 4-bit counters, then widen
                    const uint32_t n = acc[2 * u] + __shfl_xor_sync(kFull, acc[2 * u + 1], 16);
                    e1[u] = n & 0x0F0F0F0Fu;
                    o1[u] = (n >> 4) & 0x0F0F0F0Fu;
                }
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) {                 // xor 16 on 4-bit counters, widen both, add
                    const uint32_t h = __shfl_xor_sync(kFull, acc[2 * u + 1], 16);
                    e1[u] = (acc[2 * u] & 0x0F0F0F0Fu) + (h & 0x0F0F0F0Fu);
                    o1[u] = ((acc[2 * u] >> 4) & 0x0F0F0F0Fu) + ((h >> 4) & 0x0F0F0F0Fu);
                }
            }
            uint32_t w4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) w4[u] = e1[u] + __shfl_xor_sync(kFull, o1[u], 8);
            uint32_t x2[2];
            const bool b2 = lane & 4, b1 = lane & 2;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const uint32_t send = b2 ? w4[j] : w4[j + 2];
                const uint32_t keep = b2 ? w4[j + 2] : w4[j];
                x2[j] = keep + __shfl_xor_sync(kFull, send, 4);
            }
            const uint32_t v1 = (b1 ? x2[1] : x2[0]) + __shfl_xor_sync(kFull, b1 ? x2[0] : x2[1], 2);
            const uint32_t tot = (v1 & 0x00FF00FFu) + __shfl_xor_sync(kFull, (v1 >> 8) & 0x00FF00FFu, 1);
            const uint32_t col = 4 * b + red_u;
            const uint32_t c0 = tot & 0xFFFFu, c1 = tot >> 16;
#if HHT_RASTER_ATOMIC_NOZ
            atomicAdd(dst + 16 * col + red_row, c0);
            atomicAdd(dst + 16 * col + red_row + 4, c1);
#else
            if (c0) atomicAdd(dst + 16 * col + red_row, c0);
            if (c1) atomicAdd(dst + 16 * col + red_row + 4, c1);
#endif
        }
    }
};

template <typename I, bool PREF>
__global__ void __launch_bounds__(256, PREF ? 2 : 3) k_tail16(const PassArgs A) {
    // table entry e of lane copy c at slot 32e + c: an LDS.64 serves 16 lanes per wavefront and
    // every lane reads its own bank pair, so lookups never conflict whatever entries lanes need
    fill_tab16();
    __syncthreads();
    const int lane = threadIdx.x & 31;
    Raster16<I> R;
    R.init(A, lane);
    chunk_loop<PREF>(A, lane, [&](const ChunkDesc& d, const uint32_t (&p)[kItems]) {
        R.template run<kItems>(p, (int)d.cnt, d.a, d.c, d.beta, A.votes + (uint64_t)(d.r - A.nf_rbase) * kTail16Cells, lane);
    });
}

// ---------------------------------------------------------------------------------------------
// Fused tail: the pass over the lists of the split regions R at level l = D-5 and the dense 16x16
// raster of their split children (level D-4) in one kernel, without materialising level-(D-4)
// lists. A warp owns one parent R at a time (dynamic, via an atomic counter) and walks its chunks:
// each chunk's entries are tested against R's 4 children (the exact test of k_pass) and pushed onto
// per-child stacks in shared memory (4 x kQ entries per warp); whenever a stack holds a full batch
// (kFusedBatch entries), that batch from its top is rastered over that child's leaf grid exactly as k_tail16 would
// raster a chunk of the child's list (the order of a list is irrelevant to its counts); the last
// partial stacks are flushed when R is done. Entries never leave the SM between the two steps.
// ---------------------------------------------------------------------------------------------
// Block shape (C5 fused tail, one B200; build with -D to compare). With the current raster setup:
// 16 warps x 13 lines per lane (one 512-thread block per SM: one raster table per SM, 416-entry
// batches) 122.3 ms; x 12 123.8, x 11 126.4, x 10 128.3, x 14 128.3. First sweep (64-bit setup,
// two-shuffle first reduce level): 16 x 12 132.5 ms; 16 x 11 133.2,
// x 13 134.6, x 14 137.4, x 9 / x 10 137.0, x 15 141.0, x 8 141.8, x 7 140.9; 12 warps x 14 149.0;
// 8 warps x 7 (two blocks per SM, 224-entry batches, the previous default) 142.2. Loading a
// chunk's entries when it is pushed instead of one chunk ahead (HHT_FUSED_JIT, 8 registers fewer
// during the raster): 135.2 (12 lines), 139.0 (13), 141.4 (14).
#ifndef HHT_FUSED_WARPS
#define HHT_FUSED_WARPS 16                        // warps per block (1 block/SM); 8: 2 blocks/SM
#endif
#ifndef HHT_FUSED_JIT
#define HHT_FUSED_JIT 0                           // 1: load a chunk's entries when pushed, not ahead
#endif
#ifndef HHT_FUSED_BATCH_LEAN
#define HHT_FUSED_BATCH_LEAN 1                    // per-batch bookkeeping without branches or atomics (0: the old form)
#endif
#ifndef HHT_FUSED_LINEAR
#define HHT_FUSED_LINEAR 1                        // 1: chunk spans derived from the first chunk (no descriptor loads)
#endif
#ifndef HHT_FUSED_DESC_AHEAD
#define HHT_FUSED_DESC_AHEAD 0                    // 1: each chunk's list span loaded one chunk ahead
#endif
#ifndef HHT_FUSED_ITEMS
#define HHT_FUSED_ITEMS 13                        // raster batches of 13 lines per lane (416 entries)
#endif
constexpr int kFusedWarps = HHT_FUSED_WARPS;
constexpr int kFusedThreads = kWarp * kFusedWarps;
constexpr int kFusedMinBlocks = kFusedWarps <= 8 ? 2 : 1;
constexpr int kFusedItems = HHT_FUSED_ITEMS;
constexpr uint32_t kFusedBatch = kWarp * kFusedItems;
// stack capacity per child: < kFusedBatch left + <= 256 pushed (512 for 224-entry batches)
constexpr int kQ = ((int)kFusedBatch - 1 + 256 + 63) / 64 * 64;
constexpr int kFusedSmem = kFusedWarps * 4 * kQ * 4;   // dynamic: the stacks (the table is static)

template <typename I, bool GP>
__global__ void __launch_bounds__(kFusedThreads, kFusedMinBlocks) k_fused(const PassArgs A) {
    extern __shared__ uint4 s_dyn[];
    uint32_t* s_q = reinterpret_cast<uint32_t*>(s_dyn);
    fill_tab16();
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t* Q = s_q + (threadIdx.x >> 5) * (4 * kQ);
    const uint32_t q_sa = (uint32_t)__cvta_generic_to_shared(Q);
    Raster16<I> R;
    R.init(A, lane);
    const int D = A.D;
    const int sh = D - A.level;                       // == 5: parent side 32 lattice steps
    const I N = (I)A.N;
    const I Qc = ((I)3 * N) << (sh - 1);              // child b-step 3N * s/2

    while (true) {
        uint32_t u = 0;
        if (lane == 0) u = atomicAdd(A.work, 1u);
        u = __shfl_sync(kFull, u, 0);
        uint32_t r, sub = 0;
        if (A.units) {                                 // split units: (parent, block of K chunks)
            if (u >= *A.nunits) break;
            const uint2 e = __ldg(A.units + u);
            r = e.x;
            sub = e.y;
        } else {
            r = u + A.r_lo;
            if (r >= A.r_hi) break;
        }
        // the list streamed: r's own, or (tail_depth 6) its parent's, whose entries that miss r
        // get no child bits (a line crossing a child of r crosses r)
        const uint32_t lr = GP ? __ldg(A.gp_parent + r) : r;
        uint64_t c_lo = __ldg(A.p_choff + lr), c_hi = __ldg(A.p_choff + lr + 1);
        if (A.units && sub != kUnitWhole) {
            const uint64_t K = *A.unit_k;
            c_lo += (uint64_t)sub * K;
            c_hi = min(c_hi, c_lo + K);
        }
        if (c_lo >= c_hi) continue;
        // lanes 0..3: grid index of child `lane` (+ q0): its next-frontier index when only split
        // children are rastered, 4 (r - r_lo) + lane when all are; kNone for skipped children
        uint32_t my_nf = kNone;
        if (lane < 4) {
            if (A.all_children) {
                my_nf = 4 * (r - A.r_lo) + lane;
            } else {
                my_nf = __ldg(A.nf + 4 * (uint64_t)(r - A.nf_rbase) + lane);
                if (my_nf != kNone && (my_nf < A.q0 || my_nf >= A.q1)) my_nf = kNone;
            }
        }
        uint32_t nfq[4], splitm = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            nfq[q] = __shfl_sync(kFull, my_nf, q);
            splitm |= (nfq[q] != kNone ? 1u : 0u) << q;
        }
        if (splitm == 0) continue;
        ChunkDesc d = load_desc(A.chunks, c_lo, c_hi);
        const uint32_t pa = GP ? __ldg(A.gp_a + r) : d.a;
        const uint32_t pc = GP ? __ldg(A.gp_c + r) : d.c;
        const uint32_t beta = d.beta;
        const I i0 = (I)pa << sh;
        const I j0 = (I)pc << sh;
        const I alpha = ((I)1 << D) - 2 * i0;
        const I beta_m1 = (N << D) - (I)3 * N * j0 - 1;
        uint32_t top0 = 0, top1 = 0, top2 = 0, top3 = 0;   // stack heights (warp-uniform)
        uint32_t p[kItems];
#if !HHT_FUSED_JIT
        load_items(p, A.list, A.list_base, d, lane);
#endif
#if HHT_FUSED_DESC_AHEAD
        uint64_t n_e0;                                     // the next chunk's list offset and count
        uint32_t n_cnt;
        span_of(A.chunks, c_lo + 1, c_hi, n_e0, n_cnt);
#elif HHT_FUSED_LINEAR
        // a region's chunks are consecutive kChunk-entry pieces of its list (k_chunk_map), so chunk
        // ch starts kChunk (ch - c_lo) entries after chunk c_lo and holds kChunk entries except the
        // region's last: no descriptor load per chunk (the next chunk's entry loads issue at once)
        const uint32_t cnt_last =
            c_hi - c_lo > 1 ? __ldg(reinterpret_cast<const uint32_t*>(A.chunks + (c_hi - 1)) + 1) : d.cnt;
#endif
        uint64_t ch = c_lo;
        uint32_t streamed = 0;                             // entries of this work unit (profiling)
        uint32_t rastered = 0;                             // (child, line) pairs rastered (profiling)
        // One loop whose every iteration either rasters one stack (a full one, or once the parent's
        // chunks are exhausted any non-empty one) or pushes one chunk: the raster code is
        // instantiated once (four inlined copies measured 2x slower: instruction-cache misses).
        while (true) {
            const uint32_t full = (top0 >= kFusedBatch ? 1u : 0u) | (top1 >= kFusedBatch ? 2u : 0u) |
                                  (top2 >= kFusedBatch ? 4u : 0u) | (top3 >= kFusedBatch ? 8u : 0u);
            const uint32_t nonempty = (top0 ? 1u : 0u) | (top1 ? 2u : 0u) | (top2 ? 4u : 0u) | (top3 ? 8u : 0u);
            const uint32_t job = full ? full : (ch >= c_hi ? nonempty : 0u);
            if (job) {
                const int q = __ffs(job) - 1;
                const uint32_t t = q == 0 ? top0 : q == 1 ? top1 : q == 2 ? top2 : top3;
                const uint32_t n = min(t, kFusedBatch);
                const uint32_t base = t - n;               // raster the top n entries of stack q
                uint32_t pq[kFusedItems];
#if HHT_RASTER_VALID_BRANCH
                // full batches (the common case) read the stack unpredicated; slots past a partial
                // batch are zeroed (their lines are also masked inside the raster)
                if (n == kFusedBatch) {
#pragma unroll
                    for (int it = 0; it < kFusedItems; ++it) pq[it] = Q[q * kQ + base + lane + kWarp * it];
                } else {
#pragma unroll
                    for (int it = 0; it < kFusedItems; ++it)
                        pq[it] = (lane + kWarp * it < (int)n) ? Q[q * kQ + base + lane + kWarp * it] : 0u;
                }
#else
#pragma unroll
                for (int it = 0; it < kFusedItems; ++it)
                    pq[it] = (lane + kWarp * it < (int)n) ? Q[q * kQ + base + lane + kWarp * it] : 0u;
#endif
                const uint32_t nf_q = __shfl_sync(kFull, my_nf, q);
                R.template run<kFusedItems>(pq, (int)n, 2 * pa + quad_da(q), 2 * pc + quad_dc(q), beta,
                                            A.votes + (uint64_t)(nf_q - A.q0) * kTail16Cells, lane);
#if HHT_FUSED_BATCH_LEAN
                rastered += n;                             // flushed once per work unit
                top0 = q == 0 ? base : top0;               // branch-free (the if-chain compiled to branches)
                top1 = q == 1 ? base : top1;
                top2 = q == 2 ? base : top2;
                top3 = q == 3 ? base : top3;
#else
                if (lane == 0) atomicAdd(A.child_pairs, (unsigned long long)n);
                if (q == 0) top0 = base; else if (q == 1) top1 = base; else if (q == 2) top2 = base; else top3 = base;
#endif
                __syncwarp();
                continue;
            }
            if (ch >= c_hi) break;
#if HHT_FUSED_JIT
            load_items(p, A.list, A.list_base, d, lane);
#endif
            // push chunk ch: child bits of its entries (split children only)
            const int cnt = (int)d.cnt;
            streamed += (uint32_t)cnt;
            uint32_t cm = 0;
            if (GP) {
                // the parent's list: entries may miss R, so all four exact child tests
#pragma unroll
                for (int it = 0; it < kItems; ++it) {
                    const uint32_t w = p[it];
                    const I ex = (I)__byte_perm(w, 0, beta ? 0x4410u : 0x4432u);
                    const I ey = (I)__byte_perm(w, 0, beta ? 0x4432u : 0x4410u);
                    I gm1 = ex * alpha + (ey << D) + beta_m1;  // G(SW corner of R) - 1
                    if (lane + kWarp * it >= cnt) gm1 = (I)-1;
                    const I Pc = ex << sh;
                    const I Uc = Pc + Qc;
                    const uint32_t b = crosses<I>(gm1 - Pc - Qc, Uc) | (crosses<I>(gm1 - Qc, Uc) << 1) |
                                       (crosses<I>(gm1, Uc) << 2) | (crosses<I>(gm1 - Pc, Uc) << 3);
                    cm |= b << (4 * it);
                }
            } else {
                // R's own list: every entry crosses R, so y = G_SW - 1 lies in [0, 2 Uc) and the NE
                // child (G_centre > 0 >= G_NE, i.e. y >= Uc) is crossed exactly when the SW child
                // (y < Uc) is not (the SW + NE identity); SE and NW keep their exact tests. Lanes
                // past the chunk are masked once per chunk.
#pragma unroll
                for (int it = 0; it < kItems; ++it) {
                    const uint32_t w = p[it];
                    const I ex = (I)__byte_perm(w, 0, beta ? 0x4410u : 0x4432u);
                    const I ey = (I)__byte_perm(w, 0, beta ? 0x4432u : 0x4410u);
                    const I y = ex * alpha + (ey << D) + beta_m1;   // G(SW corner of R) - 1
                    const I Pc = ex << sh;
                    const I Uc = Pc + Qc;
                    const uint32_t b = (crosses<I>(y, Uc) ? 4u : 1u) | (crosses<I>(y - Qc, Uc) << 1) |
                                       (crosses<I>(y - Pc, Uc) << 3);
                    cm |= b << (4 * it);
                }
                const int nv = cnt - lane;                    // valid items of this lane: ceil(nv / 32)
                const int kv = nv <= 0 ? 0 : min((nv + kWarp - 1) / kWarp, kItems);
                cm &= kv >= kItems ? 0xFFFFFFFFu : ((1u << (4 * kv)) - 1u);
            }
            cm &= splitm * 0x11111111u;
            // push onto the stacks: byte-field warp scan of the 4 per-lane counts (as in k_pass)
            const uint32_t c0 = __popc(cm & 0x11111111u), c1 = __popc(cm & 0x22222222u);
            const uint32_t c2 = __popc(cm & 0x44444444u), c3 = __popc(cm & 0x88888888u);
            const uint32_t own = c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
            uint32_t inc = own;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                uint32_t t;
                asm volatile("{\n\t.reg .pred p;\n\tshfl.sync.up.b32 %0|p, %1, %2, 0, 0xffffffff;\n\t@!p mov.b32 %0, 0;\n\t}"
                             : "=r"(t) : "r"(inc), "r"(dd));
                inc += t;
            }
            const uint32_t exc = inc - own;
            const uint32_t t02 = __reduce_add_sync(kFull, c0 | (c2 << 16));
            const uint32_t t13 = __reduce_add_sync(kFull, c1 | (c3 << 16));
            uint32_t sa[4] = {q_sa + 4 * (top0 + (exc & 0xFFu)), q_sa + 4 * (kQ + top1 + ((exc >> 8) & 0xFFu)),
                              q_sa + 4 * (2 * kQ + top2 + ((exc >> 16) & 0xFFu)),
                              q_sa + 4 * (3 * kQ + top3 + (exc >> 24))};
#pragma unroll
            for (int it = 0; it < kItems; ++it) {
#pragma unroll
                for (int q = 0; q < 4; ++q) sts_if(cm & (1u << (4 * it + q)), sa[q], p[it]);
            }
            top0 += t02 & 0xFFFFu;
            top1 += t13 & 0xFFFFu;
            top2 += t02 >> 16;
            top3 += t13 >> 16;
            __syncwarp();
            // the next chunk's entries are in flight while the full stacks are rastered
            ++ch;
#if HHT_FUSED_DESC_AHEAD
            // the entries' addresses come from the span loaded one chunk earlier, so their loads
            // issue at once (ncu: the address add waiting on a just-issued descriptor load was the
            // fused tail's top stall site, 4 % of its samples)
            d.cnt = n_cnt;
            d.e0 = n_e0;
            span_of(A.chunks, ch + 1, c_hi, n_e0, n_cnt);
#elif HHT_FUSED_LINEAR
            d.e0 += kChunk;
            d.cnt = ch + 1 == c_hi ? cnt_last : (ch < c_hi ? (uint32_t)kChunk : 0u);
#else
            d = load_desc(A.chunks, ch, c_hi);
#endif
#if !HHT_FUSED_JIT
            load_items(p, A.list, A.list_base, d, lane);
#endif
        }
        if (lane == 0) atomicAdd(A.child_pairs + 1, (unsigned long long)streamed);
#if HHT_FUSED_BATCH_LEAN
        if (lane == 0) atomicAdd(A.child_pairs, (unsigned long long)rastered);
#else
        (void)rastered;
#endif
    }
}

// Work units of a fused-tail launch (hht_driver.cu tail_fused). With few parents (k_split == 0):
// K = max(4, ceil(chunks / target)) chunks per unit, parent r of [r_lo, r_hi) split into
// ceil(chunks_r / K) units (r, k). With many parents (k_split = K > 0): parents before r_split are
// whole units (r, kUnitWhole) and only the last ones, [r_split, r_hi), are split into units of K
// chunks, so the warps that finish last finish with small pieces. Listed in parent order. One
// block; a chunked block scan over the parents.
__global__ void __launch_bounds__(1024) k_units(const uint64_t* __restrict__ p_choff, uint32_t r_lo, uint32_t r_hi,
                                                 uint32_t target, uint32_t r_split, uint32_t k_split,
                                                 uint2* __restrict__ units, uint32_t* __restrict__ nk) {
    __shared__ uint32_t s_w[33];
    const uint64_t total = p_choff[r_hi] - p_choff[r_lo];
    const uint32_t K = k_split ? k_split : (uint32_t)max((uint64_t)4, (total + target - 1) / max(target, 1u));
    if (!k_split) r_split = r_lo;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t carry = 0;
    for (uint32_t base = r_lo; base < r_hi; base += blockDim.x) {
        const uint32_t r = base + tid;
        const uint32_t n = r >= r_hi ? 0u : r < r_split ? 1u : (uint32_t)((p_choff[r + 1] - p_choff[r] + K - 1) / K);
        uint32_t inc = n;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(kFull, inc, d);
            if (lane >= d) inc += t;
        }
        if (lane == 31) s_w[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            const uint32_t w = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0u;
            uint32_t wi = w;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t = __shfl_up_sync(kFull, wi, d);
                if (lane >= d) wi += t;
            }
            if (lane < (int)(blockDim.x >> 5)) s_w[lane] = wi - w;
            if (lane == 31) s_w[32] = wi;
        }
        __syncthreads();
        const uint32_t off = carry + s_w[wid] + inc - n;
        if (r < r_split) units[off] = make_uint2(r, kUnitWhole);
        else for (uint32_t k = 0; k < n; ++k) units[off + k] = make_uint2(r, k);
        carry += s_w[32];
        __syncthreads();
    }
    if (tid == 0) { nk[0] = carry; nk[1] = K; }
}

cudaError_t launch_units(const uint64_t* p_choff, uint32_t r_lo, uint32_t r_hi, uint32_t target_units, uint32_t r_split,
                         uint32_t k_split, uint2* units, uint32_t* nunits_k, cudaStream_t st) {
    k_units<<<1, 1024, 0, st>>>(p_choff, r_lo, r_hi, target_units, r_split, k_split, units, nunits_k);
    return cudaGetLastError();
}

int fused_blocks_per_sm(bool int64) {
    int n = 0;
    if (int64) {
        cudaFuncSetAttribute(k_fused<int64_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem);
        cudaFuncSetAttribute(k_fused<int64_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_fused<int64_t, false>, kFusedThreads, kFusedSmem);
    } else {
        cudaFuncSetAttribute(k_fused<int32_t, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem);
        cudaFuncSetAttribute(k_fused<int32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFusedSmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_fused<int32_t, false>, kFusedThreads, kFusedSmem);
    }
    return n > 0 ? n : 1;
}

cudaError_t launch_fused(bool int64, const PassArgs& a, int grid, cudaStream_t st) {
    // GP: work units stream their parents' lists (tail_depth 6); its own kernel, so the default
    // one carries a single copy of the push code (instruction cache)
    if (a.gp_parent) {
        if (int64) k_fused<int64_t, true><<<grid, kFusedThreads, kFusedSmem, st>>>(a);
        else k_fused<int32_t, true><<<grid, kFusedThreads, kFusedSmem, st>>>(a);
    } else {
        if (int64) k_fused<int64_t, false><<<grid, kFusedThreads, kFusedSmem, st>>>(a);
        else k_fused<int32_t, false><<<grid, kFusedThreads, kFusedSmem, st>>>(a);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Edge front end (§3 "Sobel's gradient operator is being
// applied", readings DESIGN.md R18-R21 after SPEC.md:104-131): per interior pixel
//   gx = sum_dy w(dy) (I(x+1, y+dy) - I(x-1, y+dy)),  gy = sum_dx w(dx) (I(x+dx, y+1) - I(x+dx, y-1))
// (w = 1, 2, 1; geometric y = H-1-row), edge iff |gx| + |gy| >= thr > 0, ALPHA iff |gx| <= |gy|,
// each set compacted in raster order. A tile of 256 threads covers 4096 consecutive pixels, lane l
// of warp w taking pixels 512w + 32k + l (coalesced byte loads); ballots give in-order positions
// within the warp, a block scan orders the warps, and a single-pass look-back over packed 64-bit
// (status | ALPHA count | BETA count) words orders the tiles, so no second pass over the image.
// ---------------------------------------------------------------------------------------------
namespace {
constexpr unsigned long long kEdgeAgg = 1ull << 62, kEdgeInc = 2ull << 62, kEdgeMask = (1ull << 31) - 1;
__device__ __forceinline__ unsigned long long edge_word(unsigned long long st, uint32_t a, uint32_t b) {
    return st | ((unsigned long long)a << 31) | (unsigned long long)b;
}
}  // namespace

__global__ void __launch_bounds__(256) k_edges(const EdgeArgs A) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_wa[8], s_wb[8];
    __shared__ uint32_t s_pa, s_pb;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(A.tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t npix = (uint64_t)A.W * A.H;
    const uint64_t p0 = (uint64_t)tile * kEdgeTile + 512 * wid + lane;
    // pixel k of this lane: p0 + 32k -> (r, c), stepped without divisions
    uint32_t r = (uint32_t)(p0 / (uint64_t)A.W), c = (uint32_t)(p0 - (uint64_t)r * A.W);
    uint32_t em = 0, am = 0;
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
        const uint64_t p = p0 + 32 * k;
        if (p < npix && A.thr > 0 && r >= 1 && r + 1 < (uint32_t)A.H && c >= 1 && c + 1 < (uint32_t)A.W) {
            const uint8_t* m = A.img + (uint64_t)r * A.W + c;
            const uint8_t* u = m - A.W;
            const uint8_t* d = m + A.W;
            const int ul = __ldg(u - 1), uc = __ldg(u), ur = __ldg(u + 1);
            const int ml = __ldg(m - 1), mr = __ldg(m + 1);
            const int dl = __ldg(d - 1), dc = __ldg(d), dr = __ldg(d + 1);
            const int gx = (ur - ul) + 2 * (mr - ml) + (dr - dl);
            const int gy = (ul + 2 * uc + ur) - (dl + 2 * dc + dr);   // row above = geometric y+1
            const int ax = abs(gx), ay = abs(gy);
            if (ax + ay >= A.thr) {
                em |= 1u << k;
                if (ax <= ay) am |= 1u << k;
            }
        }
        c += 32;
        while (c >= (uint32_t)A.W) { c -= A.W; ++r; }
    }
    // tile order: warp counts -> block scan -> look-back over tiles
    const uint32_t wa = __reduce_add_sync(kFull, __popc(em & am)), wb = __reduce_add_sync(kFull, __popc(em & ~am));
    if (lane == 0) { s_wa[wid] = wa; s_wb[wid] = wb; }
    __syncthreads();
    if (wid == 0) {
        const uint32_t va = lane < 8 ? s_wa[lane] : 0, vb = lane < 8 ? s_wb[lane] : 0;
        uint32_t ia = va, ib = vb;
#pragma unroll
        for (int dd = 1; dd < 8; dd <<= 1) {
            const uint32_t ta = __shfl_up_sync(kFull, ia, dd), tb = __shfl_up_sync(kFull, ib, dd);
            if (lane >= dd) { ia += ta; ib += tb; }
        }
        if (lane < 8) { s_wa[lane] = ia - va; s_wb[lane] = ib - vb; }
        const uint32_t ta = __shfl_sync(kFull, ia, 7), tb = __shfl_sync(kFull, ib, 7);
        using dev_u64w = cuda::atomic_ref<unsigned long long, cuda::thread_scope_device>;
        uint32_t ea = 0, eb = 0;
        if (tile == 0) {
            if (lane == 0) dev_u64w(A.tiles[0]).store(edge_word(kEdgeInc, ta, tb), cuda::memory_order_relaxed);
        } else {
            if (lane == 0) dev_u64w(A.tiles[tile]).store(edge_word(kEdgeAgg, ta, tb), cuda::memory_order_relaxed);
            int64_t pred = (int64_t)tile - 1;
            while (true) {
                const int64_t t = pred - lane;
                unsigned long long wv = kEdgeInc;                 // before tile 0: inclusive zero
                if (t >= 0) {
                    do { wv = dev_u64w(A.tiles[t]).load(cuda::memory_order_relaxed); } while ((wv >> 62) == 0);
                }
                const uint32_t pm = __ballot_sync(kFull, (wv >> 62) == 2);
                const int stop = pm ? __ffs(pm) - 1 : 31;
                uint32_t xa = (uint32_t)((wv >> 31) & kEdgeMask), xb = (uint32_t)(wv & kEdgeMask);
                if (lane > stop || t < 0) { xa = 0; xb = 0; }
                ea += __reduce_add_sync(kFull, xa);
                eb += __reduce_add_sync(kFull, xb);
                if (pm) break;
                pred -= 32;
            }
            if (lane == 0) dev_u64w(A.tiles[tile]).store(edge_word(kEdgeInc, ea + ta, eb + tb), cuda::memory_order_relaxed);
        }
        if (lane == 0) {
            s_pa = ea;
            s_pb = eb;
            if (tile == A.ntiles - 1) { A.totals[0] = ea + ta; A.totals[1] = eb + tb; }
        }
    }
    __syncthreads();
    // in-order writes: ballot per k gives each edge pixel its rank within the warp's 32 pixels
    const uint32_t lt = (1u << lane) - 1;
    uint32_t pa = s_pa + s_wa[wid], pb = s_pb + s_wb[wid];
    r = (uint32_t)(p0 / (uint64_t)A.W);
    c = (uint32_t)(p0 - (uint64_t)r * A.W);
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
        const bool e = (em >> k) & 1u, isa = e && ((am >> k) & 1u), isb = e && !((am >> k) & 1u);
        const uint32_t ba = __ballot_sync(kFull, isa), bb = __ballot_sync(kFull, isb);
        const uint32_t pt = (c << 16) | (uint32_t)(A.H - 1 - (int)r);
        if (isa) A.outA[pa + __popc(ba & lt)] = pt;
        if (isb) A.outB[pb + __popc(bb & lt)] = pt;
        pa += __popc(ba);
        pb += __popc(bb);
        c += 32;
        while (c >= (uint32_t)A.W) { c -= A.W; ++r; }
    }
}

// Rows whose width is a multiple of 16 (every power-of-two image): thread t of tile g owns the 16
// consecutive pixels 4096 g + 16 t of one row, read as one 16-byte vector per row (rows r-1, r, r+1)
// plus two halo bytes, so raster order is thread order.
// Edge (em) and ALPHA (am) bit masks of the 16 pixels starting at raster index p; r, c0 set.
// Two pixels per 32-bit word, 16 bits each (columns c and c + 2 of a 4-byte group: (0,2), (1,3),
// (4,6), ...), and the Sobel sums separably: per column s = u + 2m + d and t = u - d (u, m, d the rows
// above, at and below), gx = s[c+1] - s[c-1], gy = t[c-1] + 2 t[c] + t[c+1]. Every half carries a
// positive bias so that plain 32-bit adds never borrow across the halves: t + 256, gx + 0x4000,
// gy + 1024; |v| + bias = max(v + bias, 2 bias - (v + bias)) (VIMNMX.S16x2, values below 2^15). The
// two decisions are the top bit of each half of
//   |gx| + |gy| - thr + 0x8000   (edge: |gx| + |gy| >= thr; thr clamped to 2041 > max |gx| + |gy|)
//   |gy| - |gx| + 0x8000         (ALPHA: |gx| <= |gy|)
// ~11 instructions per pixel instead of ~45 for the per-pixel 3x3 form.
__device__ __forceinline__ void edge_masks16(const EdgeArgs& A, uint64_t p, uint32_t& r, uint32_t& c0,
                                             uint32_t& em, uint32_t& am) {
    em = am = 0;
    r = (uint32_t)(p / (uint64_t)A.W);
    c0 = (uint32_t)(p - (uint64_t)r * A.W);
    if (p >= (uint64_t)A.W * A.H || A.thr <= 0 || r < 1 || r + 1 >= (uint32_t)A.H) return;
    const uint8_t* m = A.img + (uint64_t)r * A.W + c0;
    const bool hasl = c0 > 0, hasr = c0 + 16 < (uint32_t)A.W;
    uint4 rows[3];
    uint32_t hl[3], hr[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {                 // j = 0: row above (geometric y+1), 1: this row, 2: below
        const uint8_t* q = m + (j - 1) * (int64_t)A.W;
        rows[j] = __ldg(reinterpret_cast<const uint4*>(q));
        hl[j] = hasl ? __ldg(q - 1) : 0;
        hr[j] = hasr ? __ldg(q + 16) : 0;
    }
    // S[2g], T[2g]: columns (4g, 4g+2); S[2g+1], T[2g+1]: columns (4g+1, 4g+3)
    uint32_t S[8], T[8];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        const uint32_t u = g == 0 ? rows[0].x : g == 1 ? rows[0].y : g == 2 ? rows[0].z : rows[0].w;
        const uint32_t c = g == 0 ? rows[1].x : g == 1 ? rows[1].y : g == 2 ? rows[1].z : rows[1].w;
        const uint32_t d = g == 0 ? rows[2].x : g == 1 ? rows[2].y : g == 2 ? rows[2].z : rows[2].w;
        const uint32_t ue = u & 0x00FF00FFu, ce = c & 0x00FF00FFu, de = d & 0x00FF00FFu;
        const uint32_t uo = __byte_perm(u, 0, 0x4341), co = __byte_perm(c, 0, 0x4341), dd = __byte_perm(d, 0, 0x4341);
        S[2 * g] = ue + 2 * ce + de;
        S[2 * g + 1] = uo + 2 * co + dd;
        T[2 * g] = ue - de + 0x01000100u;
        T[2 * g + 1] = uo - dd + 0x01000100u;
    }
    const uint32_t sl = hl[0] + 2 * hl[1] + hl[2], sr = hr[0] + 2 * hr[1] + hr[2];   // columns -1 and 16
    const uint32_t tl = hl[0] - hl[2] + 256u, tr = hr[0] - hr[2] + 256u;
    uint32_t E = 0, Q = 0;
    const uint32_t thr = (uint32_t)min(A.thr, 2041);
    const uint32_t ke = 0x80008000u - 0x44004400u - thr * 0x10001u;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        // left of (4g, 4g+2) = (4g-1, 4g+1); right of (4g+1, 4g+3) = (4g+2, 4g+4)
        const uint32_t Sl = g == 0 ? __byte_perm(sl, S[1], 0x5410) : __byte_perm(S[2 * g - 1], S[2 * g + 1], 0x5432);
        const uint32_t Tl = g == 0 ? __byte_perm(tl, T[1], 0x5410) : __byte_perm(T[2 * g - 1], T[2 * g + 1], 0x5432);
        const uint32_t Sr = g == 3 ? __byte_perm(S[6], sr, 0x5432) : __byte_perm(S[2 * g], S[2 * g + 2], 0x5432);
        const uint32_t Tr = g == 3 ? __byte_perm(T[6], tr, 0x5432) : __byte_perm(T[2 * g], T[2 * g + 2], 0x5432);
#pragma unroll
        for (int o = 0; o < 2; ++o) {
            // word w = 2g + o: o = 0 has neighbours (Sl, S[w+1]); o = 1 has (S[w-1], Sr)
            const uint32_t s_lo = o == 0 ? Sl : S[2 * g], s_hi = o == 0 ? S[2 * g + 1] : Sr;
            const uint32_t t_lo = o == 0 ? Tl : T[2 * g], t_hi = o == 0 ? T[2 * g + 1] : Tr;
            const uint32_t gxb = s_hi - s_lo + 0x40004000u;
            const uint32_t ax = __vmaxs2(gxb, 0x80008000u - gxb);            // |gx| + 0x4000
            const uint32_t gyb = t_lo + t_hi + 2 * T[2 * g + o];               // gy + 1024
            const uint32_t ay = __vmaxs2(gyb, 0x08000800u - gyb);            // |gy| + 1024
            const uint32_t e = ax + ay + ke, q = ay - ax + 0xBC00BC00u;
            // bit 15 -> column 4g + o, bit 31 -> bit 16 + 4g + o (column 4g + o + 2, folded below)
            const int sh = 15 - (4 * g + o);
            E |= (e >> sh) & (0x10001u << (4 * g + o));
            Q |= (q >> sh) & (0x10001u << (4 * g + o));
        }
    }
    em = (E | (E >> 14)) & 0xFFFFu;
    if (!hasl) em &= ~1u;                      // image columns 0 and W-1 have no gradient
    if (!hasr) em &= ~0x8000u;
    am = (Q | (Q >> 14)) & em;
}

// Rows whose width is a multiple of 16: two launches and no look-back. A single pass with a
// decoupled look-back over the 4096-pixel tiles (round 1) spent 45 % of its stall samples at the
// barrier behind warp 0's look-back: the ~1200 resident tiles of a wave publish their aggregates
// together and the inclusive prefix then walks them 32 per L2 round trip (ncu, round 2; one
// look-back word per warp instead was slower still, 0.26 vs 0.17 ms; a one-block scan kernel between
// the two passes cost 23 us). Here
//   k_edges16_masks  reads the image once, writes each thread's (em | am << 16) word and the tile's
//                    (ALPHA count << 32 | BETA count), and adds the latter to its super-tile's sum
//                    (2^super_shift tiles, at most 256 super-tiles: one 64-bit atomic per tile);
//   k_edges16_write  warp 0 sums the earlier super-tiles and the earlier tiles of its own super-tile
//                    (a few loads per lane, no dependence on other blocks) while the other warps
//                    reread their mask words (1/4 B per pixel) and scan them in thread (= raster)
//                    order; each warp then stages its points in shared memory (ALPHA from the front
//                    of its 512 words, BETA from the back) and copies both runs out coalesced.
__global__ void __launch_bounds__(256) k_edges16_masks(const EdgeArgs A) {
    __shared__ uint32_t s_w[8];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t tile = blockIdx.x;
    uint32_t r, c0, em, am;
    edge_masks16(A, (uint64_t)tile * kEdgeTile + 16ull * tid, r, c0, em, am);
    A.masks[(size_t)tile * 256 + tid] = em | (am << 16);
    const uint32_t w = __reduce_add_sync(kFull, __popc(em & am) | (__popc(em & ~am) << 16));
    if (lane == 0) s_w[wid] = w;
    __syncthreads();
    if (tid == 0) {
        uint32_t t = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) t += s_w[i];
        const unsigned long long c = ((unsigned long long)(t & 0xFFFFu) << 32) | (t >> 16);
        A.tiles[tile] = c;
        if (c) atomicAdd(A.supers + (tile >> A.super_shift), c);
    }
}

__global__ void __launch_bounds__(256) k_edges16_write(const EdgeArgs A) {
    __shared__ uint32_t s_w[8];
    __shared__ unsigned long long s_base;
    __shared__ uint32_t s_pts[8][512];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t tile = blockIdx.x;
    const uint32_t mw = A.masks[(size_t)tile * 256 + tid];
    if (wid == 0) {
        const uint32_t sb = tile >> A.super_shift;
        unsigned long long sum = 0;
#pragma unroll 4
        for (uint32_t i = lane; i < sb; i += 32) sum += A.supers[i];
#pragma unroll 4
        for (uint32_t t = (sb << A.super_shift) + lane; t < tile; t += 32) sum += A.tiles[t];
#pragma unroll
        for (int dd = 16; dd; dd >>= 1) sum += __shfl_xor_sync(kFull, sum, dd);
        if (lane == 0) s_base = sum;
    }
    const uint32_t em = mw & 0xFFFFu, ma = mw >> 16, mb = em & ~ma;   // am is a subset of em
    const uint32_t own = __popc(ma) | (__popc(mb) << 16);
    uint32_t inc = own;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, inc, dd);
        if (lane >= dd) inc += t;
    }
    const uint32_t wtot = __shfl_sync(kFull, inc, 31);
    if (lane == 31) s_w[wid] = inc;
    // stage: ALPHA points at s_pts[wid][0 ..), BETA points at s_pts[wid][511 ..) downwards
    {
        const uint64_t p = (uint64_t)tile * kEdgeTile + 16ull * tid;
        const uint32_t r = (uint32_t)(p / (uint64_t)A.W), c0 = (uint32_t)(p - (uint64_t)r * A.W);
        uint32_t pt = (c0 << 16) | ((uint32_t)(A.H - 1) - r);
        const uint32_t excl = inc - own;
        uint32_t* qa = &s_pts[wid][excl & 0xFFFFu];
        uint32_t* qb = &s_pts[wid][511 - (excl >> 16)];
        if (em) {
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                if ((ma >> k) & 1u) *qa++ = pt;
                if ((mb >> k) & 1u) *qb-- = pt;
                pt += 1u << 16;
            }
        }
    }
    __syncthreads();
    uint32_t before = 0;
#pragma unroll
    for (int i = 0; i < 7; ++i) before += i < wid ? s_w[i] : 0u;
    const unsigned long long tb = s_base;
    if (tid == 0 && tile == A.ntiles - 1) {
        uint32_t t = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) t += s_w[i];
        A.totals[0] = (tb >> 32) + (t & 0xFFFFu);
        A.totals[1] = (tb & 0xFFFFFFFFull) + (t >> 16);
    }
    const uint32_t na = wtot & 0xFFFFu, nb = wtot >> 16;
    uint32_t* __restrict__ oa = A.outA + ((uint32_t)(tb >> 32) + (before & 0xFFFFu));
    uint32_t* __restrict__ ob = A.outB + ((uint32_t)tb + (before >> 16));
#pragma unroll 1
    for (uint32_t i = lane; i < na; i += 32) oa[i] = s_pts[wid][i];
#pragma unroll 1
    for (uint32_t i = lane; i < nb; i += 32) ob[i] = s_pts[wid][511 - i];
}

cudaError_t launch_edges(const EdgeArgs& a, cudaStream_t st) {
    if (a.ntiles == 0) return cudaSuccess;
    if (a.W % 16 == 0) {
        k_edges16_masks<<<a.ntiles, 256, 0, st>>>(a);
        k_edges16_write<<<a.ntiles, 256, 0, st>>>(a);
    } else {
        k_edges<<<a.ntiles, 256, 0, st>>>(a);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// solution() with point removal: the removal-on result
// equals a greedy pass over the removal-off candidate leaves in depth-first order that emits a leaf
// iff its voters not yet removed exceed THRESHOLD and then removes them (live votes only shrink, so a
// leaf live at its turn had live ancestors at theirs; pinned in tests/test_oracle_removal.py).
//
// Every candidate keeps its live vote count live[c] = votes(c) - #{removed points crossing c}
// (votes(c) counts every point of the tree crossing the leaf cell, containment SURVEY.md L5). One
// cooperative kernel runs the greedy for all trees of a group at once, in rounds:
//   A  (one block per tree) the next candidate k at or after the tree's cursor with live[k] > T is
//      exact (every earlier emission's removals are applied): emit it with live votes live[k];
//   B1 (grid) every live point of the tree whose line crosses leaf k (the exact leaf test
//      0 < G_SW <= 2ex + 3N) is removed and queued, with its support pair (line, point);
//   B2 (grid, one warp per queued point) its line is rastered over the 2^D x 2^D leaf grid (column i:
//      rows f_(i+1) .. f_i with f_i = floor((G(i, 0) - 1) / 3N)) and every candidate cell it crosses
//      after k loses one live vote (a dense cell -> candidate map).
// So a round costs E tests plus the removed points' rasters; the whole post-pass is bounded by
// rounds <= E / T per tree and sum over removed points of 2^D columns (no candidates x points state).
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_rm_init(const LeafRec* __restrict__ leaves, const uint64_t* __restrict__ cand_lo,
                                                 uint32_t t0, uint32_t t1, int D, uint32_t* __restrict__ live,
                                                 uint32_t* __restrict__ cellmap) {
    const uint64_t k0 = cand_lo[t0], k1 = cand_lo[t1];
    for (uint64_t k = k0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < k1; k += (uint64_t)gridDim.x * blockDim.x) {
        const LeafRec L = leaves[k];
        live[k] = L.votes;
        const uint64_t cell = ((uint64_t)(L.tree - t0) << (2 * D)) + ((uint64_t)L.i << D) + L.j;
        cellmap[cell] = (uint32_t)(k - cand_lo[L.tree]);
    }
}

namespace cg = cooperative_groups;

// RED (at most kRmRedTrees trees in the group): every block runs A for every tree redundantly on
// identical data (no barrier between A and B1; block 0 writes the outputs), so a round costs two
// grid barriers instead of three.
template <typename I, bool RED>
__global__ void __launch_bounds__(kRmThreads) k_rm(const RmArgs A) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t s_found;
    __shared__ uint32_t s_cur[kRmRedTrees], s_pos[kRmRedTrees], s_outn[kRmRedTrees], s_fnd[kRmRedTrees];
    const uint32_t nt = A.t1 - A.t0;
    const I N = (I)A.N, N3 = (I)3 * (I)A.N;
    const int D = A.D;
    const uint32_t side = 1u << D;
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t gsize = (uint64_t)gridDim.x * blockDim.x;
    if (RED) {
        for (uint32_t tt = threadIdx.x; tt < nt; tt += blockDim.x) {
            s_cur[tt] = A.cur[A.t0 + tt];
            s_pos[tt] = A.pos[A.t0 + tt];
            s_outn[tt] = A.out_n[A.t0 + tt];
        }
        __syncthreads();
    }
    for (uint32_t round = 0;; ++round) {
        // ---- A: next emission of every active tree. RED: every block, all trees at once (thread j of
        // tree tt = threadIdx % nt scans 4 consecutive candidates per step); else block b takes trees
        // b, b + grid, ... one after another with the whole block.
        uint32_t active = 0;
        if (RED) {
            const uint32_t tt = threadIdx.x % nt, j = threadIdx.x / nt, per = blockDim.x / nt;
            const uint32_t t = A.t0 + tt;
            const uint64_t c0 = A.cand_lo[t], c1 = A.cand_lo[t + 1];
            if (threadIdx.x < nt) s_fnd[threadIdx.x] = kNone;
            __syncthreads();
            const bool mine_active = j < per && s_cur[tt] != kDone;
            for (uint64_t step = 0;; ++step) {
                const uint64_t k = c0 + s_pos[tt] + step * 4ull * per + 4ull * j;
                if (mine_active && s_fnd[tt] == kNone) {
                    uint32_t mine = kNone;
#pragma unroll
                    for (int q = 3; q >= 0; --q) {
                        const uint64_t c = k + q;
                        if (c < c1 && (uint64_t)A.live[c] > A.T) mine = (uint32_t)(c - c0);
                    }
                    if (mine != kNone) atomicMin(&s_fnd[tt], mine);
                }
                __syncthreads();
                const bool more = j == 0 && mine_active && s_fnd[tt] == kNone &&
                                  c0 + s_pos[tt] + (step + 1) * 4ull * per < c1;
                if (!__syncthreads_or(more)) break;
            }
            if (threadIdx.x < nt) {
                const uint32_t u = A.t0 + threadIdx.x, f = s_fnd[threadIdx.x];
                if (s_cur[threadIdx.x] != kDone) {
                    if (f == kNone) {
                        s_cur[threadIdx.x] = kDone;
                        if (blockIdx.x == 0) A.cur[u] = kDone;
                    } else {
                        if (blockIdx.x == 0) {
                            const uint64_t cb = A.cand_lo[u];
                            A.out[cb + s_outn[threadIdx.x]] = f;
                            A.out_live[cb + s_outn[threadIdx.x]] = A.live[cb + f];
                            A.out_n[u] = s_outn[threadIdx.x] + 1;
                            A.cur[u] = f;
                            A.pos[u] = f + 1;
                        }
                        s_cur[threadIdx.x] = f;
                        s_pos[threadIdx.x] = f + 1;
                        s_outn[threadIdx.x] += 1;
                    }
                }
            }
            __syncthreads();
            for (uint32_t q = 0; q < nt; ++q) active += s_cur[q] != kDone;
        } else {
            for (uint32_t tt = blockIdx.x; tt < nt; tt += gridDim.x) {
                const uint32_t t = A.t0 + tt;
                if (A.cur[t] == kDone) continue;
                const uint64_t c0 = A.cand_lo[t], c1 = A.cand_lo[t + 1];
                uint32_t found = kNone;
                // 4 consecutive candidates per thread per step; one barrier per step until one is live
                for (uint64_t k = c0 + A.pos[t]; k < c1; k += 4ull * blockDim.x) {
                    uint32_t mine = kNone;
#pragma unroll
                    for (int j = 3; j >= 0; --j) {
                        const uint64_t c = k + 4ull * threadIdx.x + j;
                        if (c < c1 && (uint64_t)A.live[c] > A.T) mine = (uint32_t)(c - c0);
                    }
                    if (__syncthreads_or(mine != kNone)) {
                        if (threadIdx.x == 0) s_found = kNone;
                        __syncthreads();
                        if (mine != kNone) atomicMin(&s_found, mine);
                        __syncthreads();
                        found = s_found;
                        __syncthreads();
                        break;
                    }
                }
                if (threadIdx.x == 0) {
                    if (found == kNone) {
                        A.cur[t] = kDone;
                    } else {
                        const uint32_t e = A.out_n[t];
                        A.out[c0 + e] = found;
                        A.out_live[c0 + e] = A.live[c0 + found];
                        A.out_n[t] = e + 1;
                        A.cur[t] = found;
                        A.pos[t] = found + 1;
                        atomicAdd(A.active + (round & 1), 1u);
                    }
                }
            }
        }
        if (gtid == 0) { A.active[(round + 1) & 1] = 0; A.qn[(round + 1) & 1] = 0; }
        if (RED) {
            if (active == 0) break;                // identical in every block
        } else {
            grid.sync();
            if (A.active[round & 1] == 0) break;
        }
        uint32_t* qn = A.qn + (round & 1);
        uint32_t* queue = A.queue + (round & 1) * 2 * (uint64_t)A.queue_cap;
        // ---- B1: remove the live voters of every tree's emitted leaf. RED (few trees): the grid
        // strides over each tree's points; else block b takes trees b, b + grid, ...
        for (uint32_t tt = RED ? 0 : blockIdx.x; tt < nt; tt += RED ? 1 : gridDim.x) {
            const uint32_t t = A.t0 + tt;
            const uint32_t k = RED ? s_cur[tt] : A.cur[t];
            if (k == kDone) continue;
            const uint32_t slot = (uint32_t)(A.cand_lo[t] + (RED ? s_outn[tt] : A.out_n[t]) - 1);   // global line slot
            const LeafRec L = A.leaves[A.cand_lo[t] + k];
            const bool beta = A.tree_beta[t] != 0;
            const uint32_t n = A.pt_n[t];
            const uint32_t* pts = A.packed + A.pt_off[t];
            uint8_t* rem = A.removed + A.rm_off[t];
            const I base = (N << D) - N3 * (I)L.j;
            const uint64_t p0 = RED ? gtid : threadIdx.x, ps = RED ? gsize : blockDim.x;
            for (uint64_t p = p0; p < n; p += ps) {
                if (rem[p]) continue;
                const uint32_t pk = pts[p];
                const I ex = (I)(beta ? (pk & 0xFFFFu) : (pk >> 16)), ey = (I)(beta ? (pk >> 16) : (pk & 0xFFFFu));
                const I g = base + ((ex + ey) << D) - (I)2 * (I)L.i * ex;      // G(SW corner of leaf k)
                if (g > 0 && g <= (I)2 * ex + N3) {
                    rem[p] = 1;
                    const uint32_t q = atomicAdd(qn, 1u);
                    queue[2 * (uint64_t)q] = t;
                    queue[2 * (uint64_t)q + 1] = (uint32_t)p;
                    const unsigned long long sidx = atomicAdd(A.sup_n, 1ull);
                    A.sup[2 * sidx] = slot;
                    A.sup[2 * sidx + 1] = (uint32_t)p;
                }
            }
        }
        grid.sync();
        // ---- B2: every queued point's line loses one live vote in every later candidate it crosses;
        // one thread per (queued point, run of kRmCols leaf columns): rows f_(i+1) .. f_i of column i,
        // f_i = floor((G(i, 0) - 1) / 3N) with the remainder carried column to column (2ex < 3N: at
        // most one borrow per column); all cell-map loads of a run are issued before its atomics
        const uint32_t nq = *qn;
        const uint32_t runs = (side + kRmCols - 1) / kRmCols;
        const uint64_t work = (uint64_t)nq * runs;
        for (uint64_t wi = gtid; wi < work; wi += gsize) {
            const uint32_t qi = (uint32_t)(wi / runs), run = (uint32_t)(wi - (uint64_t)qi * runs);
            const uint32_t t = queue[2 * (uint64_t)qi], p = queue[2 * (uint64_t)qi + 1];
            const uint32_t k = RED ? s_cur[t - A.t0] : A.cur[t];
            const bool beta = A.tree_beta[t] != 0;
            const uint32_t pk = A.packed[A.pt_off[t] + p];
            const I ex = (I)(beta ? (pk & 0xFFFFu) : (pk >> 16)), ey = (I)(beta ? (pk >> 16) : (pk & 0xFFFFu));
            const uint32_t i_lo = run * kRmCols;
            I y = ((ex + ey + N) << D) - (I)2 * (I)i_lo * ex - 1;   // G(i_lo, 0) - 1
            I f, r;
            if (y >= 0) { f = y / N3; r = y - f * N3; }
            else { f = -((-y + N3 - 1) / N3); r = y - f * N3; }
            const uint32_t* cm = A.cellmap + ((uint64_t)(t - A.t0) << (2 * D));
            uint32_t* live = A.live + A.cand_lo[t];
            uint32_t c0[kRmCols], c1[kRmCols];
#pragma unroll
            for (int u = 0; u < kRmCols; ++u) {
                I rn = r - (I)2 * ex, fn = f;
                if (rn < 0) { rn += N3; fn -= 1; }
                const uint32_t i = i_lo + u;
                const I vlo = fn < 0 ? (I)0 : fn, vhi = f >= (I)side ? (I)side - 1 : f;
                // rows vlo .. vhi hold 0, 1 or 2 cells (f drops by at most one per column)
                const bool ok0 = i < side && vlo <= vhi, ok1 = ok0 && vhi > vlo;
                const uint64_t col = (uint64_t)i << D;
                c0[u] = ok0 ? __ldg(cm + col + (uint64_t)vlo) : kNone;
                c1[u] = ok1 ? __ldg(cm + col + (uint64_t)vhi) : kNone;
                f = fn;
                r = rn;
            }
#pragma unroll
            for (int u = 0; u < kRmCols; ++u) {
                if (c0[u] != kNone && c0[u] > k) atomicSub(live + c0[u], 1u);
                if (c1[u] != kNone && c1[u] > k) atomicSub(live + c1[u], 1u);
            }
        }
        grid.sync();
    }
}

// Compact the emitted lines into hht_leaf rows (image, half, i, j, live) in tree order and the
// supports into (line index, point) pairs: slot k = cand_lo[t] + e is line line_base[t] + e.
__device__ __forceinline__ uint32_t rm_tree_of(const uint64_t* cand_lo, uint32_t nt, uint64_t k) {
    uint32_t lo = 0, hi = nt - 1;                 // last t with cand_lo[t] <= k
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) / 2;
        if (cand_lo[mid] <= k) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(256) k_rm_rows(const LeafRec* __restrict__ leaves, const uint64_t* __restrict__ cand_lo,
                                                 const uint32_t* __restrict__ out, const uint32_t* __restrict__ out_live,
                                                 const uint32_t* __restrict__ out_n, const uint64_t* __restrict__ line_base,
                                                 const uint8_t* __restrict__ tree_beta, uint32_t nt, uint32_t H,
                                                 uint64_t ncand, uint32_t* __restrict__ rows,
                                                 uint32_t* __restrict__ sup, uint64_t nsup) {
    const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gs = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = g; k < ncand; k += gs) {
        const uint32_t t = rm_tree_of(cand_lo, nt, k);
        const uint64_t e = k - cand_lo[t];
        if (e >= out_n[t]) continue;
        const LeafRec L = leaves[cand_lo[t] + out[k]];
        uint32_t* r = rows + 5 * (line_base[t] + e);
        r[0] = t / H;
        r[1] = tree_beta[t] ? 2u : 1u;
        r[2] = L.i;
        r[3] = L.j;
        r[4] = out_live[k];
    }
    for (uint64_t s = g; s < nsup; s += gs) {
        const uint32_t slot = sup[2 * s];
        const uint32_t t = rm_tree_of(cand_lo, nt, slot);
        sup[2 * s] = (uint32_t)(line_base[t] + (slot - cand_lo[t]));
    }
}

cudaError_t launch_rm_rows(const LeafRec* leaves, const uint64_t* cand_lo, const uint32_t* out, const uint32_t* out_live,
                           const uint32_t* out_n, const uint64_t* line_base, const uint8_t* tree_beta, uint32_t nt,
                           uint32_t H, uint64_t ncand, uint32_t* rows, uint32_t* sup, uint64_t nsup, cudaStream_t st) {
    k_rm_rows<<<148 * 8, 256, 0, st>>>(leaves, cand_lo, out, out_live, out_n, line_base, tree_beta, nt, H, ncand, rows,
                                       sup, nsup);
    return cudaGetLastError();
}

int rm_blocks_per_sm(bool int64) {
    int n = 0, m = 0;
    if (int64) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_rm<int64_t, false>, kRmThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, k_rm<int64_t, true>, kRmThreads, 0);
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_rm<int32_t, false>, kRmThreads, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, k_rm<int32_t, true>, kRmThreads, 0);
    }
    n = std::min(n, m);
    return n > 0 ? n : 1;
}

cudaError_t launch_removal(const RmArgs& a, const LeafRec* leaves, bool int64, int grid, cudaStream_t st) {
    k_rm_init<<<1184, 256, 0, st>>>(leaves, a.cand_lo, a.t0, a.t1, a.D, a.live, a.cellmap);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    void* args[] = {(void*)&a};
    const bool red = a.t1 - a.t0 <= (uint32_t)kRmRedTrees;
    const void* fn = int64 ? (red ? (const void*)k_rm<int64_t, true> : (const void*)k_rm<int64_t, false>)
                           : (red ? (const void*)k_rm<int32_t, true> : (const void*)k_rm<int32_t, false>);
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kRmThreads), args, 0, st);
}

// ---------------------------------------------------------------------------------------------
// Latency path: a detection whose lists are tiny (the paper's own image sizes) runs as ONE launch of
// one 1024-thread block that walks every level itself, so a single image costs one kernel instead of
// ~30 launches and ~10 host synchronisations. Same method and outputs as the multi-kernel path: at
// each level, one pass over the (region, candidate) pairs counts the 4 child votes with the exact
// test (0 < G_SW <= s (2ex + 3N), PAPER.md:85 / DESIGN.md §4), a block scan over the children writes
// their records and the next frontier (strict votes > T) or the leaves at level D, and a
// second pass appends each candidate to the lists of the split children it crosses.
// ---------------------------------------------------------------------------------------------
// frontier tree ids carry the tree's half in their top bit: no global load per region in the passes
constexpr uint32_t kSmallBeta = 1u << 31;

#ifdef HHT_SMALL_TRACE
// phase timestamps of the last k_small launch (experiment builds only: scripts/build_variant.sh)
__device__ unsigned long long g_small_trace[512];
#define SMALL_MARK(k) do { if (threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_small_trace[k] = t_; } } while (0)
extern "C" int hht_debug_small_trace(unsigned long long* host) {
    return (int)cudaMemcpyFromSymbol(host, g_small_trace, sizeof g_small_trace);
}
#else
#define SMALL_MARK(k) do { } while (0)
#endif

template <typename I>
__global__ void __launch_bounds__(1024) k_small(const SmallArgs A) {
    __shared__ uint32_t s_warp[33], s_warp2[33];
    __shared__ uint32_t s_F;
    __shared__ unsigned long long s_v[32], s_sv[32];
    // every per-level array lives in shared memory (the host admits only problems that fit), so the
    // dependent phases of a level cost shared-memory, not L2, round trips
    extern __shared__ uint4 s_small_dyn[];
    // layout: [list 0 | list 1] (unless the host gave device buffers: global_scratch), then per
    // buffer b = 0, 1 the frontier arrays tree | a | c | off of FS = smem_F + 1 entries each, then the
    // child votes and the children's frontier indices. Buffers are addressed as base + b * stride, so
    // nothing indexes a pointer array with the level parity (that would live in local memory)
    uint32_t* w = reinterpret_cast<uint32_t*>(s_small_dyn);
    const uint32_t Sm = A.smem_S, FS = A.smem_F + 1;
    uint32_t* list0 = A.list[0];
    if (!A.global_scratch) { list0 = w; w += 2 * Sm; }
    uint32_t* const fr = w;                              // frontier buffer 0, buffer 1 at fr + 4 FS
    uint32_t* const cv = fr + 8 * FS;                    // [4 F] child votes
    uint32_t* const cursor = cv + 4 * (FS - 1);          // [4 F] split child's frontier index or kNone
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const I N = (I)A.N;
    const int D = A.D;
    unsigned long long my_v = 0, my_t = 0;              // this thread's share of the votes and tests
    SMALL_MARK(0);
    for (uint32_t i = tid; i < kStatCount; i += blockDim.x) A.stats[i] = 0;   // the call's statistics start at 0
    for (uint32_t i = tid; i < (uint32_t)D + 2; i += blockDim.x) A.counts[i] = 0;   // levels never reached stay 0
    // K0 in the same launch: stage and range-check the points (an out-of-range point fails
    // the call before any traversal; the host reads the flag with the results)
    if (A.pts) {
        uint32_t bad = 0;
        for (uint64_t i = tid; i < A.npts; i += blockDim.x) {
            const int2 p = A.pts[i];
            const bool ok = (unsigned)p.x < (unsigned)A.N && (unsigned)p.y < (unsigned)A.N;
            bad |= !ok;
            A.packed[i] = ok ? (((uint32_t)p.x << 16) | (uint32_t)p.y) : 0u;
        }
        if (__syncthreads_or(bad)) {
            if (tid == 0) {
                A.fin[0] = 1;
                __threadfence_system();
            }
            return;
        }
    }
    // level 0: roots (every line crosses the root); split iff E > T (reading R6)
    if (tid == 0) {
        uint32_t F = 0, S = 0;
        for (uint32_t t = 0; t < A.ntrees; ++t) {
            const uint32_t E = A.tree_n[t];
            A.rec[0][t] = {t, 0, 0, E};
            my_t += E;
            my_v += E;
            if ((uint64_t)E > A.T) {
                fr[F] = t | (A.tree_beta[t] ? kSmallBeta : 0u);
                fr[FS + F] = 0;
                fr[2 * FS + F] = 0;
                fr[3 * FS + F] = S;
                S += E;
                ++F;
                my_t += 4ull * E;                         // the root's 4 child tests per point
            }
        }
        fr[3 * FS + F] = S;
        A.counts[0] = A.ntrees;
        s_F = F;
    }
    __syncthreads();
    if (tid == 0) {                                       // after the zeroing above
        A.stats[kStatVisited0] = A.ntrees;
        A.stats[kStatSplit0] = s_F;
    }
    // root lists: the trees' points, in frontier order
    for (uint32_t r = 0; r < s_F; ++r) {
        const uint32_t t = fr[r] & ~kSmallBeta, o = fr[3 * FS + r], n = A.tree_n[t];
        const uint32_t* src = A.packed + A.tree_off[t];
        for (uint32_t i = tid; i < n; i += blockDim.x) list0[o + i] = src[i];
    }
    __syncthreads();
    SMALL_MARK(1);
    for (int l = 0; l < D; ++l) {
        const uint32_t F = s_F;
        if (F == 0) break;
        const uint32_t cur = (uint32_t)l & 1u;
        const uint32_t* const list = list0 + cur * Sm;
        uint32_t* const nlist = list0 + (cur ^ 1u) * Sm;
        const uint32_t* const ftree = fr + cur * 4 * FS;
        const uint32_t* const fa = ftree + FS;
        const uint32_t* const fc = ftree + 2 * FS;
        const uint32_t* const off = ftree + 3 * FS;
        uint32_t* const ntree = fr + (cur ^ 1u) * 4 * FS;
        const int sh = D - l;
        const I Qc = ((I)3 * N) << (sh - 1);
        SMALL_MARK(8 + 8 * l);
        // pass 1 (level 0 only; deeper levels get their child votes from the previous level's pass 2):
        // child votes. A warp owns whole regions (their pairs are contiguous in the list): the region's
        // data is loaded once, no search per pair, and the warp sums the 4 child votes itself
        if (l == 0) {
            for (uint32_t r = wid; r < F; r += nw) {
                const bool beta = (ftree[r] & kSmallBeta) != 0;
                const I i0 = (I)fa[r] << sh, j0 = (I)fc[r] << sh;
                const I alpha = ((I)1 << D) - 2 * i0, gb = (N << D) - (I)3 * N * j0;
                uint32_t v0 = 0, v1 = 0, v2 = 0, v3 = 0;
                for (uint32_t i = off[r] + lane; i < off[r + 1]; i += 32) {
                    const uint32_t p = list[i];
                    const I ex = (I)(beta ? (p & 0xFFFFu) : (p >> 16)), ey = (I)(beta ? (p >> 16) : (p & 0xFFFFu));
                    const I g = ex * alpha + (ey << D) + gb;   // G(SW)
                    const I Pc = ex << sh, Uc = Pc + Qc;
                    // children NE, NW, SW, SE: SW values g - Pc - Qc, g - Qc, g, g - Pc
                    v0 += g - Pc - Qc > 0 && g - Pc - Qc <= Uc;
                    v1 += g - Qc > 0 && g - Qc <= Uc;
                    v2 += g > 0 && g <= Uc;
                    v3 += g - Pc > 0 && g - Pc <= Uc;
                }
                v0 = __reduce_add_sync(0xFFFFFFFFu, v0);
                v1 = __reduce_add_sync(0xFFFFFFFFu, v1);
                v2 = __reduce_add_sync(0xFFFFFFFFu, v2);
                v3 = __reduce_add_sync(0xFFFFFFFFu, v3);
                if (lane == 0) { cv[4 * r] = v0; cv[4 * r + 1] = v1; cv[4 * r + 2] = v2; cv[4 * r + 3] = v3; }
            }
            __syncthreads();
        }
        SMALL_MARK(9 + 8 * l);
        // children, in one block scan of (split flag, split ? votes : 0): records of all, the next
        // frontier with its list offsets (or the leaves at level D), and each child's frontier index
        const bool leaf = l + 1 == D;
        Record* const rec = A.rec[l + 1];
        uint32_t nf = 0, S2 = 0;                         // running totals of the scan
        for (uint32_t base = 0; base < 4 * F; base += blockDim.x) {
            const uint32_t k = base + tid, r = k >> 2, q = k & 3;
            const bool ok = k < 4 * F;
            const uint32_t v = ok ? cv[k] : 0u;
            const bool split = ok && (uint64_t)v > A.T;
            uint32_t tr = 0, ca = 0, cb = 0;
            if (ok) {
                tr = ftree[r];
                ca = 2 * fa[r] + quad_da((int)q);
                cb = 2 * fc[r] + quad_dc((int)q);
                rec[k] = {tr & ~kSmallBeta, ca, cb, v};
                my_v += v;
                if (split && !leaf) my_t += 4ull * v;      // 4 code evaluations per voter of a split region
            }
            uint32_t in = split ? 1u : 0u, is = split ? v : 0u;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t tn = __shfl_up_sync(0xFFFFFFFFu, in, d), ts = __shfl_up_sync(0xFFFFFFFFu, is, d);
                if (lane >= d) { in += tn; is += ts; }
            }
            if (lane == 31) { s_warp[wid] = in; s_warp2[wid] = is; }
            __syncthreads();
            if (wid == 0) {
                const uint32_t wn = lane < nw ? s_warp[lane] : 0u, ws = lane < nw ? s_warp2[lane] : 0u;
                uint32_t xn = wn, xs = ws;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t tn = __shfl_up_sync(0xFFFFFFFFu, xn, d), ts = __shfl_up_sync(0xFFFFFFFFu, xs, d);
                    if (lane >= d) { xn += tn; xs += ts; }
                }
                if (lane < nw) { s_warp[lane] = xn - wn; s_warp2[lane] = xs - ws; }
                if (lane == 31) { s_warp[32] = xn; s_warp2[32] = xs; }
            }
            __syncthreads();
            const uint32_t f = nf + s_warp[wid] + in - 1;  // this child's frontier index when split
            if (split) {
                if (leaf) {
                    A.leaves[f] = {tr & ~kSmallBeta, ca, cb, v};
                } else {
                    ntree[f] = tr;
                    ntree[FS + f] = ca;
                    ntree[2 * FS + f] = cb;
                    ntree[3 * FS + f] = S2 + s_warp2[wid] + is - v;
                }
            }
            if (ok && !leaf) cursor[k] = split ? f : kNone;
            nf += s_warp[32];
            S2 += s_warp2[32];
            __syncthreads();                               // s_warp reuse; frontier complete for pass 2
        }
        SMALL_MARK(10 + 8 * l);
        if (tid == 0) {
            A.counts[l + 1] = 4 * F;
            A.stats[kStatVisited0 + l + 1] = 4ull * F;
            if (leaf) {
                A.counts[D + 1] = nf;
                A.stats[kStatLeaves] = nf;
            } else {
                A.stats[kStatSplit0 + l + 1] = nf;
                ntree[3 * FS + nf] = S2;
                s_F = nf;
            }
        }
        if (leaf) break;
        // pass 2: append each candidate to the lists of the split children it crosses and count, as it
        // goes, the votes of those children's own 4 children (the next level's pass 1). A warp owns
        // whole regions, so it alone writes their split children's lists and votes: positions from
        // ballots and running counts, no atomics. Per-lane grandchild counts are packed two per word
        // (a lane sees at most 1/32 of a region's list, and lists here are far below 2^21 entries) and
        // unpacked before the warp sums them
        {
            const I Qc1 = ((I)3 * N) << (sh - 2);          // the child level's Q (sh >= 2 here)
            const uint32_t* const noff = ntree + 3 * FS;
            for (uint32_t r = wid; r < F; r += nw) {
                const bool beta = (ftree[r] & kSmallBeta) != 0;
                const I i0 = (I)fa[r] << sh, j0 = (I)fc[r] << sh;
                const I alpha = ((I)1 << D) - 2 * i0, gb = (N << D) - (I)3 * N * j0;
                const uint4 fq4 = *reinterpret_cast<const uint4*>(cursor + 4 * r);
                const uint32_t fq[4] = {fq4.x, fq4.y, fq4.z, fq4.w};
                uint32_t pos[4], c01[4], c23[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    pos[q] = fq[q] != kNone ? noff[fq[q]] : 0u;
                    c01[q] = c23[q] = 0;
                }
                const uint32_t e = off[r + 1];
                for (uint32_t i = off[r] + lane; i - lane < e; i += 32) {
                    const bool ok = i < e;
                    const uint32_t p = ok ? list[i] : 0u;
                    const I ex = (I)(beta ? (p & 0xFFFFu) : (p >> 16)), ey = (I)(beta ? (p >> 16) : (p & 0xFFFFu));
                    const I g = ex * alpha + (ey << D) + gb;
                    const I Pc = ex << sh, Uc = Pc + Qc;
                    const I Pc1 = ex << (sh - 1), Uc1 = Pc1 + Qc1;
                    const I gq[4] = {g - Pc - Qc, g - Qc, g, g - Pc};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const bool app = ok && fq[q] != kNone && gq[q] > 0 && gq[q] <= Uc;
                        const uint32_t b = __ballot_sync(0xFFFFFFFFu, app);
                        if (app) {
                            nlist[pos[q] + __popc(b & ((1u << lane) - 1u))] = p;
                            const I h = gq[q];                 // G(SW) of child q: its children as in pass 1
                            c01[q] += (h - Pc1 - Qc1 > 0 && h - Pc1 - Qc1 <= Uc1 ? 1u : 0u) |
                                      (h - Qc1 > 0 && h - Qc1 <= Uc1 ? 0x10000u : 0u);
                            c23[q] += (h > 0 && h <= Uc1 ? 1u : 0u) | (h - Pc1 > 0 && h - Pc1 <= Uc1 ? 0x10000u : 0u);
                        }
                        pos[q] += __popc(b);
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (fq[q] == kNone) continue;            // warp-uniform
                    const uint32_t x0 = __reduce_add_sync(0xFFFFFFFFu, c01[q] & 0xFFFFu);
                    const uint32_t x1 = __reduce_add_sync(0xFFFFFFFFu, c01[q] >> 16);
                    const uint32_t x2 = __reduce_add_sync(0xFFFFFFFFu, c23[q] & 0xFFFFu);
                    const uint32_t x3 = __reduce_add_sync(0xFFFFFFFFu, c23[q] >> 16);
                    if (lane == 0) *reinterpret_cast<uint4*>(cv + 4 * fq[q]) = make_uint4(x0, x1, x2, x3);
                }
            }
        }
        __syncthreads();
        SMALL_MARK(14 + 8 * l);
    }
    SMALL_MARK(7);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        my_v += __shfl_xor_sync(0xFFFFFFFFu, my_v, d);
        my_t += __shfl_xor_sync(0xFFFFFFFFu, my_t, d);
    }
    if (lane == 0) { s_v[wid] = my_v; s_sv[wid] = my_t; }
    __syncthreads();
    if (tid == 0) {
        unsigned long long votes = 0, tests = 0;
        for (uint32_t i = 0; i < nw; ++i) { votes += s_v[i]; tests += s_sv[i]; }
        A.stats[kStatTests] = tests;
        A.stats[kStatVotes] = votes;
    }
    // results in the same launch: counts and statistics straight into the mapped host block (fin)
    __syncthreads();
    if (A.fin) {
        for (uint32_t i = tid; i < (uint32_t)D + 2; i += blockDim.x) A.fin[1 + i] = A.counts[i];
        unsigned long long* hs = reinterpret_cast<unsigned long long*>(A.fin + kFinishStatsWord);
        for (uint32_t i = tid; i < kStatCount; i += blockDim.x) hs[i] = A.stats[i];
        if (tid == 0) A.fin[0] = 0;
        __threadfence_system();
    }
}

// S is rounded up to a multiple of 4 entries (the host passes smem_S rounded): 16-byte aligned votes and
// frontier indices after the two lists
uint64_t small_smem_bytes(uint32_t S, uint32_t F) { return 4ull * (2ull * ((S + 3ull) & ~3ull) + 8ull * (F + 1) + 8ull * F); }
uint64_t small_frontier_bytes(uint32_t F) { return 4ull * (8ull * (F + 1) + 8ull * F); }

cudaError_t launch_small(const SmallArgs& a, bool int64, cudaStream_t st) {
    const int smem = (int)(a.global_scratch ? small_frontier_bytes(a.smem_F) : small_smem_bytes(a.smem_S, a.smem_F));
    // the dynamic shared-memory opt-in is raised only when a call needs more than any before on this
    // device (one attribute call per growth, not per launch)
    static int opted[2][64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int& have = opted[int64 ? 1 : 0][dev & 63];
    if (smem > have) {
        const cudaError_t e = int64 ? cudaFuncSetAttribute(k_small<int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)
                                    : cudaFuncSetAttribute(k_small<int32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        have = smem;
    }
    if (int64)
        k_small<int64_t><<<1, 1024, smem, st>>>(a);
    else
        k_small<int32_t><<<1, 1024, smem, st>>>(a);
    return cudaGetLastError();
}

using PassKernel = void (*)(const PassArgs);

static PassKernel tail16_kernel(bool int64, bool pref) {
    if (int64) return pref ? k_tail16<int64_t, true> : k_tail16<int64_t, false>;
    return pref ? k_tail16<int32_t, true> : k_tail16<int32_t, false>;
}

int tail16_blocks_per_sm(bool int64, bool pref) {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, tail16_kernel(int64, pref), 256, 0);
    return n > 0 ? n : 1;
}

cudaError_t launch_tail16(bool int64, bool pref, const PassArgs& a, int grid, cudaStream_t st) {
    tail16_kernel(int64, pref)<<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

int tail_blocks_per_sm(bool int64) {
    int n = 0;
    if (int64) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_tail<int64_t>, 256, 0);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_tail<int32_t>, 256, 0);
    return n > 0 ? n : 1;
}

cudaError_t launch_tail(bool int64, const PassArgs& a, int grid, cudaStream_t st) {
    if (int64) k_tail<int64_t><<<grid, 256, 0, st>>>(a);
    else k_tail<int32_t><<<grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

// Gather the 4 child votes of each parent at level c-1 from the leaf grid (side G = 2^tk leaves) of
// its ancestor at the tail level L = c-1-hops: a child region of side 2^j leaves (j = D - c) has
// votes = sum of its 2^j diagonal leaf counts (diagonal identity, see the tail kernels).
__global__ void __launch_bounds__(256) k_gather(const uint32_t* __restrict__ dense, uint32_t anc_base,
                                                const uint32_t* __restrict__ anc_a, const uint32_t* __restrict__ anc_c,
                                                const uint32_t* __restrict__ p_a, const uint32_t* __restrict__ p_c,
                                                GatherChain chain, int hops, int tk, int j, uint32_t Fp,
                                                uint32_t* __restrict__ V, const uint32_t* __restrict__ owner_parent) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= Fp) return;
    uint32_t A = p;
    for (int h = 0; h < hops; ++h) A = chain.parent[h][A];
    const uint32_t la = p_a[p] - (anc_a[A] << hops), lc = p_c[p] - (anc_c[A] << hops);
    const uint32_t G = 1u << tk, S = 1u << j;
    // grid of owner A: A - anc_base, or (all-children fused tail) 4 (parent(A) - anc_base) + quad(A)
    const uint32_t gi = owner_parent ? 4 * (owner_parent[A] - anc_base) + quad_of(anc_a[A] & 1, anc_c[A] & 1)
                                     : A - anc_base;
    const uint32_t* g = dense + (uint64_t)gi * (G * G);   // leaf grid, [G*u + v]
    uint32_t v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const uint32_t u0 = (2 * la + quad_da(q)) * S, w0 = (2 * lc + quad_dc(q)) * S;
        uint32_t sum = 0;
        for (uint32_t t = 0; t < S; ++t) sum += g[G * (u0 + t) + w0 + t];
        v[q] = sum;
    }
    reinterpret_cast<uint4*>(V)[p] = make_uint4(v[0], v[1], v[2], v[3]);
}

cudaError_t launch_gather(const uint32_t* dense, uint32_t anc_base, const uint32_t* anc_a, const uint32_t* anc_c,
                          const uint32_t* p_a, const uint32_t* p_c, const GatherChain& chain, int hops, int tk,
                          int j, uint32_t Fp, uint32_t* V, const uint32_t* owner_parent, cudaStream_t st) {
    if (Fp == 0) return cudaSuccess;
    k_gather<<<(Fp + 255) / 256, 256, 0, st>>>(dense, anc_base, anc_a, anc_c, p_a, p_c, chain, hops, tk, j, Fp, V,
                                               owner_parent);
    return cudaGetLastError();
}

// Votes of the 4 children of each of nparents parents from their own 16x16 leaf grids (grid 4p + q):
// a region's votes are the sum of its diagonal leaves (identity 2 applied recursively).
__global__ void __launch_bounds__(256) k_grid_diag(const uint32_t* __restrict__ dense, uint32_t nparents,
                                                   uint32_t* __restrict__ V) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= 4 * nparents) return;
    const uint32_t* d = dense + (uint64_t)g * kTail16Cells;
    uint32_t s = 0;
#pragma unroll
    for (int t = 0; t < 16; ++t) s += d[17 * t];
    V[g] = s;
}

cudaError_t launch_grid_diag(const uint32_t* dense, uint32_t nparents, uint32_t* V, cudaStream_t st) {
    if (nparents == 0) return cudaSuccess;
    k_grid_diag<<<(4 * nparents + 255) / 256, 256, 0, st>>>(dense, nparents, V);
    return cudaGetLastError();
}

// Chunk bounds and streamed pairs of a parent range [r0, r1) (one thread).
__global__ void k_bounds(const uint64_t* off, const uint64_t* choff, const uint32_t* len, uint32_t r0, uint32_t r1,
                         int is_root, RangeInfo* info, uint64_t* chunk_bounds, RangeInfo* info_h) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint64_t pairs = 0;
    if (is_root) {
        for (uint32_t r = r0; r < r1; ++r) pairs += len[r];
    } else {
        pairs = off[r1] - off[r0];
    }
    info->pairs = pairs;
    info->chunk_lo = chunk_bounds[0] = choff[r0];
    info->chunk_hi = chunk_bounds[1] = choff[r1];
    if (info_h) *info_h = *info;      // mapped host copy: read after a stream sync, no copy engine
}

__global__ void k_set_bounds(uint64_t* b, uint64_t lo, uint64_t hi) {
    if (threadIdx.x == 0) { b[0] = lo; b[1] = hi; }
}

cudaError_t launch_set_bounds(uint64_t* bounds, uint64_t lo, uint64_t hi, cudaStream_t st) {
    k_set_bounds<<<1, 32, 0, st>>>(bounds, lo, hi);
    return cudaGetLastError();
}

cudaError_t launch_bounds(const uint64_t* off, const uint64_t* choff, const uint32_t* len, uint32_t r0, uint32_t r1,
                          int is_root, RangeInfo* info, uint64_t* chunk_bounds, RangeInfo* info_h, cudaStream_t st) {
    k_bounds<<<1, 32, 0, st>>>(off, choff, len, r0, r1, is_root, info, chunk_bounds, info_h);
    return cudaGetLastError();
}

// n words device -> mapped host memory (small readbacks that must not queue behind bulk copies on
// the copy engines, e.g. the leaf-sink transfers).
__global__ void k_copy_u32(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

cudaError_t launch_copy_u32(uint32_t* dst, const uint32_t* src, uint32_t n, cudaStream_t st) {
    k_copy_u32<<<1, 32, 0, st>>>(dst, src, n);
    return cudaGetLastError();
}

// Leaf records (tree, i, j, votes) -> the ABI's hht_leaf rows (image, half, i, j, votes). Each warp
// converts 32 consecutive records and writes their 32 x 20 bytes as five fully coalesced 128-byte
// stores through a warp-private shared-memory transpose (stride-5 words: conflict-free both ways);
// five scattered 4-byte stores per row had touched 20 sectors per store instruction.
__global__ void __launch_bounds__(256) k_leaf_rows(const LeafRec* __restrict__ in, uint64_t n,
                                                   const uint8_t* __restrict__ tree_beta, uint32_t H,
                                                   uint32_t* __restrict__ out) {
    __shared__ uint32_t s_rows[8][5 * 32];
    const int lane = threadIdx.x & 31;
    uint32_t* sw = s_rows[threadIdx.x >> 5];
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; 32 * w < n; w += nw) {
        const uint64_t k = 32 * w + lane;
        if (k < n) {
            const LeafRec r = in[k];
            sw[5 * lane + 0] = r.tree / H;
            sw[5 * lane + 1] = tree_beta[r.tree] ? 2u : 1u;
            sw[5 * lane + 2] = r.i;
            sw[5 * lane + 3] = r.j;
            sw[5 * lane + 4] = r.votes;
        }
        __syncwarp();
        const uint64_t words = 5 * min((uint64_t)32, n - 32 * w);
        uint32_t* o = out + 160 * w;
#pragma unroll
        for (int q = 0; q < 5; ++q)
            if ((uint64_t)(lane + 32 * q) < words) o[lane + 32 * q] = sw[lane + 32 * q];
        __syncwarp();
    }
}

// Leaf records -> packed 8-byte rows (hht_set_leaf_sink_packed): i << 48 | j << 32 | votes (depth <= 16).
__global__ void __launch_bounds__(256) k_leaf_packed(const LeafRec* __restrict__ in, uint64_t n,
                                                     unsigned long long* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += stride) {
        const LeafRec r = in[k];
        out[k] = ((unsigned long long)r.i << 48) | ((unsigned long long)r.j << 32) | r.votes;
    }
}

cudaError_t launch_leaf_packed(const LeafRec* in, uint64_t n, uint64_t* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_leaf_packed<<<(unsigned)blocks, 256, 0, st>>>(in, n, reinterpret_cast<unsigned long long*>(out));
    return cudaGetLastError();
}

// Per-tree leaf offsets: out[t] = first leaf record of tree >= t (records are in tree order), t = 0..ntrees.
__global__ void __launch_bounds__(256) k_tree_offsets(const LeafRec* __restrict__ in, uint64_t n, uint32_t ntrees,
                                                      unsigned long long* __restrict__ out) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntrees) return;
    uint64_t lo = 0, hi = n;                      // lower bound of tree t
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (in[mid].tree < t) lo = mid + 1; else hi = mid;
    }
    out[t] = lo;
}

cudaError_t launch_tree_offsets(const LeafRec* in, uint64_t n, uint32_t ntrees, uint64_t* out, cudaStream_t st) {
    k_tree_offsets<<<(ntrees + 1 + 255) / 256, 256, 0, st>>>(in, n, ntrees, reinterpret_cast<unsigned long long*>(out));
    return cudaGetLastError();
}

cudaError_t launch_leaf_rows(const LeafRec* in, uint64_t n, const uint8_t* tree_beta, uint32_t H, uint32_t* out,
                             cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_leaf_rows<<<(unsigned)blocks, 256, 0, st>>>(in, n, tree_beta, H, out);
    return cudaGetLastError();
}

// The count-ahead pass keeps the register prefetch under mode 3: its bulk-copy loop needs 73 registers
// (3 blocks/SM), measured slower (C5 list passes 43.4 vs 39.7 ms with both passes on the ring)
#ifndef PF_WRITE_TMA
#define PF_WRITE_TMA 1
#endif
template <typename I, int P, int C>
static PassKernel pass_kernel_t(int mode) {
    if (mode == MODE_COUNT) return k_pass<I, MODE_COUNT, P == 2 ? 1 : P, C>;
    if (mode == MODE_WRITE) return k_pass<I, MODE_WRITE, P == 2 ? PF_WRITE_TMA : P, C>;
    if (mode == MODE_WRITE_NC && !C) return k_pass<I, MODE_WRITE_NC, P, 0>;
    return k_pass<I, MODE_COUNT2, P == 2 ? 1 : P, C>;
}

// pf: 0 = descriptor prefetch only, 1 = also the next chunk's entries in registers, 2 = bulk-copy ring
// (list passes MODE_WRITE / MODE_WRITE_NC; the other modes use 1). The circumcircle variants (1:
// lattice units, 2: (m, b) units) are instantiated with the register prefetch only.
static PassKernel pass_kernel(int mode, bool int64, int pf, int circle = 0) {
    if (circle == 1) return int64 ? pass_kernel_t<int64_t, 1, 1>(mode) : pass_kernel_t<int32_t, 1, 1>(mode);
    if (circle == 2) return int64 ? pass_kernel_t<int64_t, 1, 2>(mode) : pass_kernel_t<int32_t, 1, 2>(mode);
    if (int64) return pf == 2 ? pass_kernel_t<int64_t, 2, 0>(mode) : pf ? pass_kernel_t<int64_t, 1, 0>(mode) : pass_kernel_t<int64_t, 0, 0>(mode);
    return pf == 2 ? pass_kernel_t<int32_t, 2, 0>(mode) : pf ? pass_kernel_t<int32_t, 1, 0>(mode) : pass_kernel_t<int32_t, 0, 0>(mode);
}

static int pass_dyn_smem(int mode, int pf, int circle) {
    return (pf == 2 && !circle && (mode == MODE_WRITE_NC || (mode == MODE_WRITE && PF_WRITE_TMA == 2)))
               ? 8 * (int)kTmaWarpBytes : 0;
}

int pass_blocks_per_sm(int mode, bool int64, int pf, int circle) {
    int n = 0;
    const PassKernel k = pass_kernel(mode, int64, pf, circle);
    const int dyn = pass_dyn_smem(mode, pf, circle);
    if (dyn) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 256, dyn);
    return n > 0 ? n : 1;
}

cudaError_t launch_pass(int mode, bool int64, int pf, int circle, const PassArgs& a, int grid, cudaStream_t st) {
    pass_kernel(mode, int64, pf, circle)<<<grid, 256, pass_dyn_smem(mode, pf, circle), st>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// K3: threshold-and-split (PAPER.md:122-134 step 13: "if level.vote > THRESHOLD ... if level =
// ceil(log2 N) then solution() else level <- level+1") for every child of a range of parents.
// One thread per parent (its 4 children in quad order, a 16-byte vector load); a single-pass
// decoupled look-back scan over (split count, local list entries, chunks) gives each split child
// its next-frontier index, list offset and chunk offset in the paper's depth-first order (children
// of a parent are consecutive, parents keep their order). Writes the (key, votes) record of every
// child, the next frontier (SoA), and at the leaf level the detected lines.
// ---------------------------------------------------------------------------------------------
namespace {

struct Agg {
    uint32_t F, C;
    uint64_t S;
};

__device__ __forceinline__ Agg agg_add(Agg x, Agg y) { return {x.F + y.F, x.C + y.C, x.S + y.S}; }

__device__ __forceinline__ Agg shfl_up_agg(Agg v, int d) {
    Agg o;
    o.F = __shfl_up_sync(kFull, v.F, d);
    o.C = __shfl_up_sync(kFull, v.C, d);
    o.S = __shfl_up_sync(kFull, v.S, d);
    return o;
}

__device__ __forceinline__ Agg warp_inclusive(Agg v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Agg o = shfl_up_agg(v, d);
        if (lane >= d) v = agg_add(v, o);
    }
    return v;
}

__device__ __forceinline__ Agg warp_total(Agg v) {
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        v.F += __shfl_xor_sync(kFull, v.F, d);
        v.C += __shfl_xor_sync(kFull, v.C, d);
        v.S += __shfl_xor_sync(kFull, v.S, d);
    }
    return v;
}

using dev_u32 = cuda::atomic_ref<uint32_t, cuda::thread_scope_device>;
using dev_u64 = cuda::atomic_ref<uint64_t, cuda::thread_scope_device>;

__device__ __forceinline__ void publish(TileDesc* t, Agg v, uint32_t status) {
    if (status == 1) {
        dev_u32(t->aggF).store(v.F, cuda::memory_order_relaxed);
        dev_u32(t->aggC).store(v.C, cuda::memory_order_relaxed);
        dev_u64(t->aggS).store(v.S, cuda::memory_order_relaxed);
    } else {
        dev_u32(t->incF).store(v.F, cuda::memory_order_relaxed);
        dev_u32(t->incC).store(v.C, cuda::memory_order_relaxed);
        dev_u64(t->incS).store(v.S, cuda::memory_order_relaxed);
    }
    dev_u32(t->status).store(status, cuda::memory_order_release);
}

}  // namespace

// Persistent blocks walk the tiles (pass 0: in the order a device counter hands them out, so every
// tile a look-back waits on is held by a running block; passes 1-2: strided); the per-block vote /
// leaf / test statistics are flushed with one set of atomics per block instead of per tile.
__global__ void __launch_bounds__(kSplitThreads) k_split(const SplitArgs A) {
    __shared__ Agg s_warp[kSplitThreads / 32];
    __shared__ Agg s_prefix;
    __shared__ uint32_t s_tile;
    __shared__ uint4 s_rec[kSplitThreads / 32][128];   // per-warp record staging (4 per parent, swizzled)
    __shared__ uint4 s_leaf[kSplitThreads / 32][128];  // per-warp leaf staging (leaf level)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned long long st_votes = 0, st_split = 0, st_tests = 0, st_visited = 0;   // lane-0 partials

    for (uint32_t iter = 0;; ++iter) {
        if (tid == 0) s_tile = A.pass == 0 ? atomicAdd(A.tile_counter, 1u) : blockIdx.x + iter * gridDim.x;
        __syncthreads();
        const uint32_t tile = s_tile;
        if (tile >= A.ntiles) break;
        const uint32_t p = tile * kSplitThreads + tid;
        const bool valid = p < A.Fp;

        uint4 V = make_uint4(0, 0, 0, 0), VL = V;
        uint32_t tree = 0, pa = 0, pc = 0;
        if (valid) {
            V = __ldg(reinterpret_cast<const uint4*>(A.V) + p);
            VL = (A.VL == A.V) ? V : __ldg(reinterpret_cast<const uint4*>(A.VL) + p);
            if (A.pass != 1) {
                tree = __ldg(A.p_tree + p);
                pa = __ldg(A.p_a + p);
                pc = __ldg(A.p_c + p);
            }
        }
        if (valid && A.derive_ne) {   // votes(parent) = votes(SW child) + votes(NE child)
            V.x = __ldg(A.p_votes + p) - V.z;
            VL.x = __ldg(A.p_len + p) - VL.z;
        }
        const uint32_t v[4] = {V.x, V.y, V.z, V.w};
        const uint32_t vl[4] = {VL.x, VL.y, VL.z, VL.w};
        uint32_t flag[4], len[4], nch[4];
        Agg mine = {0, 0, 0};
        unsigned long long my_votes = 0, my_tests = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            flag[q] = (valid && (uint64_t)v[q] > A.T) ? 1u : 0u;          // strict: votes > THRESHOLD
            len[q] = (flag[q] && A.need_lists) ? vl[q] : 0u;   // list entries on this rank
            nch[q] = (len[q] + kChunk - 1) / kChunk;
            mine.F += flag[q];
            mine.C += nch[q];
            mine.S += len[q];
            my_votes += v[q];
            if (flag[q]) my_tests += 4ull * v[q];
        }

        // block scan
        const Agg incl = warp_inclusive(mine, lane);
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            Agg w = lane < kSplitThreads / 32 ? s_warp[lane] : Agg{0, 0, 0};
            const Agg wi = warp_inclusive(w, lane);
            if (lane < kSplitThreads / 32) s_warp[lane] = {wi.F - w.F, wi.C - w.C, wi.S - w.S};  // exclusive
            const Agg block_total = {__shfl_sync(kFull, wi.F, 31), __shfl_sync(kFull, wi.C, 31), shfl_u64(wi.S, 31)};
            Agg excl = {0, 0, 0};
            if (A.pass == 1) {                            // aggregates only (k_split_scan orders the tiles)
                if (lane == 0) {
                    A.tiles[tile].aggF = block_total.F;
                    A.tiles[tile].aggC = block_total.C;
                    A.tiles[tile].aggS = block_total.S;
                }
            } else if (A.pass == 2) {                     // the exclusive tile prefix is precomputed
                excl = {A.tiles[tile].incF, A.tiles[tile].incC, A.tiles[tile].incS};
            } else if (tile == 0) {
                // decoupled look-back (warp-wide window of 32 predecessors)
                if (lane == 0) publish(A.tiles + 0, block_total, 2);
            } else {
                if (lane == 0) publish(A.tiles + tile, block_total, 1);
                int64_t pred = (int64_t)tile - 1;
                while (true) {
                    const int64_t t = pred - lane;
                    uint32_t st = 2;
                    Agg val = {0, 0, 0};
                    if (t >= 0) {
                        TileDesc* d = A.tiles + t;
                        // relaxed spin (no L1 invalidation per poll), then one acquire fence: the
                        // payload was stored before the status with release semantics
                        do { st = dev_u32(d->status).load(cuda::memory_order_relaxed); } while (st == 0);
                        cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
                        if (st == 1) {
                            val = {dev_u32(d->aggF).load(cuda::memory_order_relaxed),
                                   dev_u32(d->aggC).load(cuda::memory_order_relaxed),
                                   dev_u64(d->aggS).load(cuda::memory_order_relaxed)};
                        } else {
                            val = {dev_u32(d->incF).load(cuda::memory_order_relaxed),
                                   dev_u32(d->incC).load(cuda::memory_order_relaxed),
                                   dev_u64(d->incS).load(cuda::memory_order_relaxed)};
                        }
                    }
                    const uint32_t pm = __ballot_sync(kFull, st == 2);
                    const int stop = pm ? __ffs(pm) - 1 : 31;    // nearest predecessor with a prefix
                    if (lane > stop) val = {0, 0, 0};
                    excl = agg_add(excl, warp_total(val));
                    if (pm) break;
                    pred -= 32;
                }
                if (lane == 0) publish(A.tiles + tile, agg_add(excl, block_total), 2);
            }
            if (lane == 0) {
                s_prefix = excl;
                if (A.pass == 0 && tile == A.ntiles - 1) {
                    const Agg tot = agg_add(excl, block_total);
                    A.totals->F = tot.F;
                    A.totals->S = tot.S;
                    A.totals->C = tot.C;
                    if (!A.leaf_level) {
                        A.out.off[tot.F] = tot.S;
                        A.out.choff[tot.F] = tot.C;
                    }
                }
            }
        }
        __syncthreads();
        if (A.pass != 1) {
            const Agg base = agg_add(agg_add(s_prefix, s_warp[wid]), Agg{incl.F - mine.F, incl.C - mine.C, incl.S - mine.S});

            // the warp's leaves are the contiguous range [f_w, f_w + n_w): staged, then stored coalesced
            const uint32_t f_w = __shfl_sync(kFull, base.F, 0);
            // record (lane, q) at slot 4 lane + (q ^ ((lane >> 1) & 3)): for each q the 32 lanes' 16-byte
            // stores hit 8 distinct bank groups per quarter-warp (conflict-free)
            const uint32_t swz = (lane >> 1) & 3;
            if (valid) {
                uint32_t f = base.F, cc = base.C;
                uint64_t s = base.S;
                uint32_t nf4[4];
                uint64_t so[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t ca = 2 * pa + quad_da(q), cb = 2 * pc + quad_dc(q);
                    nf4[q] = kNone;
                    so[q] = s;
                    if (flag[q]) {
                        if (A.leaf_level) {
                            s_leaf[wid][f - f_w] = make_uint4(tree, ca, cb, v[q]);
                        } else {
                            nf4[q] = f;
                            A.out.tree[f] = tree;
                            A.out.a[f] = ca;
                            A.out.c[f] = cb;
                            A.out.parent[f] = A.parent_base + p;
                            if (A.write_off) {               // read only at list levels / D-1
                                A.out.len[f] = vl[q];
                                A.out.votes[f] = v[q];
                                A.out.off[f] = s;
                                A.out.choff[f] = cc;
                            }
                        }
                        f += 1;
                        s += len[q];
                        cc += nch[q];
                    }
                    if (A.record) s_rec[wid][4 * lane + (q ^ swz)] = make_uint4(tree, ca, cb, v[q]);
                }
                if (!A.leaf_level) {
                    if (A.nf) reinterpret_cast<uint4*>(A.nf)[p] = make_uint4(nf4[0], nf4[1], nf4[2], nf4[3]);
                    if (A.need_lists) {
                        ulonglong2* o = reinterpret_cast<ulonglong2*>(A.nfoff + 4 * (uint64_t)p);
                        o[0] = make_ulonglong2(so[0], so[1]);
                        o[1] = make_ulonglong2(so[2], so[3]);
                    }
                }
            }
            if (A.record) {
                // the warp's 4 x 32 records (2 KB, contiguous in HBM) go out as fully coalesced 16-byte stores
                __syncwarp();
                const uint32_t p0 = tile * kSplitThreads + wid * 32;
                const uint32_t nrec = p0 < A.Fp ? 4 * min(32u, A.Fp - p0) : 0;
                uint4* dst = reinterpret_cast<uint4*>(A.rec) + 4 * (uint64_t)p0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t k = lane + 32 * i;             // record k: parent k / 4, quad k % 4
                    const uint32_t slot = (k & ~3u) + ((k & 3u) ^ (((k >> 2) >> 1) & 3u));
                    if (k < nrec) dst[k] = s_rec[wid][slot];
                }
            }
            if (A.leaf_level) {
                __syncwarp();
                const uint32_t n_w = __shfl_sync(kFull, base.F + mine.F, 31) - f_w;
                uint4* dst = reinterpret_cast<uint4*>(A.leaves) + f_w;
                for (uint32_t k = lane; k < n_w; k += 32) dst[k] = s_leaf[wid][k];
            }

            // stats (lane 0 of every warp keeps the warp's running partials)
            unsigned long long sv = my_votes, sf = mine.F, stt = my_tests;
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) {
                sv += __shfl_xor_sync(kFull, sv, d);
                sf += __shfl_xor_sync(kFull, sf, d);
                stt += __shfl_xor_sync(kFull, stt, d);
            }
            st_votes += sv;
            st_split += sf;
            st_tests += stt;
            if (wid == 0) {
                const uint64_t t0 = (uint64_t)tile * kSplitThreads;
                st_visited += 4ull * ((A.Fp > t0) ? min((uint64_t)kSplitThreads, (uint64_t)A.Fp - t0) : 0);
            }
        }
        __syncthreads();   // s_tile, s_warp, s_prefix and the stages are reused by the next tile
    }
    if (A.pass != 1 && lane == 0) {
        if (st_votes) atomicAdd(A.stats + kStatVotes, st_votes);
        if (A.leaf_level) {
            if (st_split) atomicAdd(A.stats + kStatLeaves, st_split);
        } else {
            if (st_split) atomicAdd(A.stats + kStatSplit0 + A.child_level, st_split);
            if (st_tests) atomicAdd(A.stats + kStatTests, st_tests);
        }
        if (st_visited) atomicAdd(A.stats + kStatVisited0 + A.child_level, st_visited);
    }
}

// Exclusive scan of the tile aggregates of pass 1 into tiles[t].inc*, totals and sentinels, by
// kScanBlocks resident blocks: block b owns a contiguous segment of tiles, reduces it (coalesced),
// gets its segment prefix from a warp-wide decoupled look-back over the earlier segments (all blocks
// are resident: the grid is at most one block per SM), then scans its segment in 1024-tile steps.
// (One block did this at ~10 MB of aggregates per C4 leaf-level split: 0.52 ms, bound by one SM's
// bandwidth.)
__device__ __forceinline__ Agg block_total_agg(Agg v, Agg* s_w) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const Agg w = warp_total(v);
    if (lane == 0) s_w[wid] = w;
    __syncthreads();
    Agg t = {0, 0, 0};
    if (wid == 0) {
        t = lane < (int)(blockDim.x >> 5) ? s_w[lane] : Agg{0, 0, 0};
        t = warp_total(t);
        if (lane == 0) s_w[32] = t;
    }
    __syncthreads();
    t = s_w[32];
    __syncthreads();
    return t;
}

__global__ void __launch_bounds__(1024) k_split_scan(const SplitArgs A, TileDesc* seg_desc) {
    __shared__ Agg s_w[33];
    __shared__ Agg s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t nseg = gridDim.x, seg = (A.ntiles + nseg - 1) / nseg;
    const uint32_t t0 = min(A.ntiles, blockIdx.x * seg), t1 = min(A.ntiles, t0 + seg);
    // 1. segment aggregate
    Agg mine = {0, 0, 0};
    for (uint32_t t = t0 + tid; t < t1; t += blockDim.x)
        mine = agg_add(mine, Agg{__ldg(&A.tiles[t].aggF), __ldg(&A.tiles[t].aggC), __ldg(&A.tiles[t].aggS)});
    const Agg segtot = block_total_agg(mine, s_w);
    // 2. segment prefix: decoupled look-back over the earlier segments (warp 0)
    if (wid == 0) {
        Agg excl = {0, 0, 0};
        if (blockIdx.x == 0) {
            if (lane == 0) publish(seg_desc, segtot, 2);
        } else {
            if (lane == 0) publish(seg_desc + blockIdx.x, segtot, 1);
            int64_t pred = (int64_t)blockIdx.x - 1;
            while (true) {
                const int64_t t = pred - lane;
                uint32_t st = 2;
                Agg val = {0, 0, 0};
                if (t >= 0) {
                    TileDesc* d = seg_desc + t;
                    do { st = dev_u32(d->status).load(cuda::memory_order_relaxed); } while (st == 0);
                    cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
                    if (st == 1) val = {dev_u32(d->aggF).load(cuda::memory_order_relaxed), dev_u32(d->aggC).load(cuda::memory_order_relaxed),
                                        dev_u64(d->aggS).load(cuda::memory_order_relaxed)};
                    else val = {dev_u32(d->incF).load(cuda::memory_order_relaxed), dev_u32(d->incC).load(cuda::memory_order_relaxed),
                                dev_u64(d->incS).load(cuda::memory_order_relaxed)};
                }
                const uint32_t pm = __ballot_sync(kFull, st == 2);
                const int stop = pm ? __ffs(pm) - 1 : 31;
                if (lane > stop) val = {0, 0, 0};
                excl = agg_add(excl, warp_total(val));
                if (pm) break;
                pred -= 32;
            }
            if (lane == 0) publish(seg_desc + blockIdx.x, agg_add(excl, segtot), 2);
        }
        if (lane == 0) {
            s_prefix = excl;
            if (blockIdx.x == nseg - 1) {
                const Agg tot = agg_add(excl, segtot);
                A.totals->F = tot.F;
                A.totals->S = tot.S;
                A.totals->C = tot.C;
                if (!A.leaf_level) {
                    A.out.off[tot.F] = tot.S;
                    A.out.choff[tot.F] = tot.C;
                }
            }
        }
    }
    __syncthreads();
    // 3. the segment's exclusive tile prefixes, 1024 tiles per step
    Agg carry = s_prefix;
    for (uint32_t base = t0; base < t1; base += blockDim.x) {
        const uint32_t t = base + tid;
        Agg a = {0, 0, 0};
        if (t < t1) a = {__ldg(&A.tiles[t].aggF), __ldg(&A.tiles[t].aggC), __ldg(&A.tiles[t].aggS)};
        const Agg incl = warp_inclusive(a, lane);
        if (lane == 31) s_w[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const Agg w = lane < (int)(blockDim.x >> 5) ? s_w[lane] : Agg{0, 0, 0};
            const Agg wi = warp_inclusive(w, lane);
            if (lane < (int)(blockDim.x >> 5)) s_w[lane] = {wi.F - w.F, wi.C - w.C, wi.S - w.S};
            if (lane == 31) s_w[32] = wi;
        }
        __syncthreads();
        if (t < t1) {
            const Agg wb = s_w[wid];
            A.tiles[t].incF = carry.F + wb.F + incl.F - a.F;
            A.tiles[t].incC = carry.C + wb.C + incl.C - a.C;
            A.tiles[t].incS = carry.S + wb.S + incl.S - a.S;
        }
        carry = agg_add(carry, s_w[32]);
        __syncthreads();
    }
}

int split_blocks_per_sm() {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_split, kSplitThreads, 0);
    return n > 0 ? n : 1;
}

cudaError_t launch_split(const SplitArgs& a, int resident_blocks, cudaStream_t st) {
    if (a.ntiles == 0) return cudaSuccess;
    const unsigned grid = a.ntiles < (uint32_t)resident_blocks ? a.ntiles : (unsigned)resident_blocks;
    if (a.ntiles < kSplitPrescanTiles) {
        SplitArgs b = a;
        b.pass = 0;
        k_split<<<grid, kSplitThreads, 0, st>>>(b);
        return cudaGetLastError();
    }
    // reduce-then-scan: with many tiles the look-back's first wave walks back over ~1000 running
    // tiles and holds their warps at the barrier; two passes over V cost 16 B per parent more
    SplitArgs b = a;
    b.pass = 1;
    k_split<<<grid, kSplitThreads, 0, st>>>(b);
    const uint32_t nseg = std::min<uint32_t>(kScanBlocks, (a.ntiles + 1023) / 1024);
    cudaMemsetAsync(a.scan_seg, 0, nseg * sizeof(TileDesc), st);
    k_split_scan<<<nseg, 1024, 0, st>>>(b, a.scan_seg);
    b.pass = 2;
    k_split<<<grid, kSplitThreads, 0, st>>>(b);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Chunk map: chunk -> region for a frontier. A persistent grid of W warps: with F >= W regions
// each warp walks regions wid, wid + W, ...; with fewer regions (the first levels: 2 root regions
// of 62.5k chunks each on C5) each region gets wpr = W / F warps that interleave its chunks 16 at
// a time, so a few huge lists do not leave one warp writing them alone (one warp per region had
// cost 130-350 us per launch at levels 0-2 of C5).
// ---------------------------------------------------------------------------------------------
constexpr unsigned kChunkMapBlocks = 148 * 8;
__global__ void __launch_bounds__(256) k_chunk_map(const uint64_t* __restrict__ choff, const uint64_t* __restrict__ off,
                                                   const uint32_t* __restrict__ len, const uint32_t* __restrict__ ra,
                                                   const uint32_t* __restrict__ rc, const uint32_t* __restrict__ tree,
                                                   const uint8_t* __restrict__ tree_beta, uint32_t F, uint32_t wpr,
                                                   ChunkDesc* __restrict__ chunks) {
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t W = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    // lane pair (2i, 2i+1) writes the two 16-byte halves of one descriptor: every store instruction
    // covers 16 consecutive descriptors (512 contiguous bytes, whole sectors)
    const uint32_t half = (uint32_t)lane & 1u;
    const uint32_t part = wpr > 1 ? wid % wpr : 0u;
    const uint32_t rstep = wpr > 1 ? W / wpr : W;
    for (uint32_t w = wpr > 1 ? wid / wpr : wid; w < F; w += rstep) {
        const uint64_t b = choff[w], e = choff[w + 1], o = off[w];
        const uint32_t n = len[w], a = ra[w], c = rc[w], beta = tree_beta[tree[w]];
        for (uint64_t k = b + 16 * (uint64_t)part + (lane >> 1); k < e; k += 16 * (uint64_t)wpr) {
            const uint64_t j = (k - b) * kChunk;
            uint4* q = reinterpret_cast<uint4*>(chunks + k) + half;
            if (half == 0) {
                const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, (uint64_t)n - j);
                *q = make_uint4(w, cnt, a, c);
            } else {
                const uint64_t e0 = o + j;
                *q = make_uint4((uint32_t)e0, (uint32_t)(e0 >> 32), beta, 0u);
            }
        }
    }
}

cudaError_t launch_chunk_map(const uint64_t* choff, const uint64_t* off, const uint32_t* len, const uint32_t* a,
                             const uint32_t* c, const uint32_t* tree, const uint8_t* tree_beta, uint32_t F,
                             ChunkDesc* chunks, cudaStream_t st) {
    if (F == 0) return cudaSuccess;
    const uint32_t W = kChunkMapBlocks * 256 / 32;
    const uint32_t wpr = F >= W ? 1u : W / F;
    k_chunk_map<<<kChunkMapBlocks, 256, 0, st>>>(choff, off, len, a, c, tree, tree_beta, F, wpr, chunks);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Range selection: largest q1 with off[q1] - off[q0] <= cap (at least q0+1), and the chunk range
// of the parents of [q0, q1). One thread; binary search.
// ---------------------------------------------------------------------------------------------
__global__ void k_range(const uint64_t* c_off, const uint32_t* c_parent, uint32_t Fc, uint32_t q0,
                        uint64_t cap, uint64_t forced_q1, const uint64_t* p_off, const uint64_t* p_choff,
                        const uint32_t* p_len, int p_is_root, RangeInfo* info, uint64_t* chunk_bounds,
                        RangeInfo* info_h) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint64_t base = c_off[q0];
    uint64_t q1;
    if (forced_q1) {
        q1 = forced_q1;
    } else {
        uint64_t lo = q0 + 1, hi = Fc;     // answer in [q0+1, Fc]
        if (c_off[hi] - base <= cap) {
            lo = hi;
        } else {
            while (lo < hi) {              // largest x in [lo, hi) with c_off[x] - base <= cap
                const uint64_t mid = (lo + hi + 1) / 2;
                if (c_off[mid] - base <= cap) lo = mid; else hi = mid - 1;
            }
        }
        q1 = lo;
    }
    const uint32_t plo = c_parent[q0], phi = c_parent[q1 - 1];
    info->q1 = q1;
    info->s_lo = base;
    info->s_hi = c_off[q1];
    info->chunk_lo = p_choff[plo];
    info->chunk_hi = p_choff[phi + 1];
    if (p_is_root) {        // root lists alias the image slices: off[] is not a scan of len[]
        uint64_t s = 0;
        for (uint32_t r = plo; r <= phi; ++r) s += p_len[r];
        info->pairs = s;
    } else {
        info->pairs = p_off[phi + 1] - p_off[plo];
    }
    chunk_bounds[0] = info->chunk_lo;
    chunk_bounds[1] = info->chunk_hi;
    if (info_h) *info_h = *info;      // mapped host copy: read after a stream sync, no copy engine
}

cudaError_t launch_range(const uint64_t* c_off, const uint32_t* c_parent, uint32_t Fc, uint32_t q0,
                         uint64_t cap_entries, uint64_t forced_q1, const uint64_t* p_off,
                         const uint64_t* p_choff, const uint32_t* p_len, int p_is_root, RangeInfo* info,
                         uint64_t* chunk_bounds, RangeInfo* info_h, cudaStream_t st) {
    k_range<<<1, 32, 0, st>>>(c_off, c_parent, Fc, q0, cap_entries, forced_q1, p_off, p_choff, p_len,
                              p_is_root, info, chunk_bounds, info_h);
    return cudaGetLastError();
}

}  // namespace hht

// Level driver and C ABI of libhht.so (declared in include/hht.h).
//
// Control flow of one detection (paper: PAPER.md:73-138 run level-synchronously):
//   K0 stage/validate -> roots (every line crosses the root, votes = E) -> count pass over the
//   roots' lists (level-1 votes) -> [allreduce] -> split(level 1) -> descend(0):
//     descend(l): for each depth-first range of the level-(l+1) frontier whose candidate lists fit
//       the memory budget: write pass over the level-l lists (compacts the level-(l+1) lists and
//       counts level-(l+2) votes) -> [allreduce] -> split(level l+2) -> descend(l+1).
//     At level D-2 the pass is count-only (level-D votes) -> split(level D) emits the leaves.
// One host synchronisation per split (the next frontier's size sizes the next launch).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <atomic>
#include <condition_variable>
#include <mutex>
#include <cmath>

#include "hht.h"
#include "hht_internal.h"

using namespace hht;

namespace {

struct Buf {
    void* p = nullptr;
    size_t cap = 0;
    uint64_t gen = 0;             // allocation generation (h2d_cached: a reallocation invalidates)
};

struct Level {
    Buf tree, a, c, parent, len, votes_g, off, choff, chunks;   // frontier R_l
    Buf nf, nfoff;                                            // children of R_(l-1) range -> R_l
    Buf votes, votes_local;                                   // votes of R_l's children (range)
    Buf cursor;                                               // append cursors of R_l lists (range)
    Buf list_own;                                             // R_l candidate lists (range)
    uint32_t F = 0;
    uint64_t S = 0, C = 0;
    const uint32_t* list = nullptr;
    uint64_t list_base = 0;

    Frontier frontier() {
        return {(uint32_t*)tree.p, (uint32_t*)a.p, (uint32_t*)c.p, (uint32_t*)parent.p, (uint32_t*)len.p,
                (uint32_t*)votes_g.p, (uint64_t*)off.p, (uint64_t*)choff.p, (ChunkDesc*)chunks.p};
    }
};

struct Grow {          // append-only device vector
    Buf b;
    uint64_t n = 0;
};

struct ProfEv {
    cudaEvent_t a, b;
    int cls;
    uint64_t bytes;
    uint64_t ops;
};

}  // namespace

// In-process collective group: `world` contexts, one host thread each. An allreduce stages every
// rank's buffer in host memory, waits for all ranks, reduces in rank order and copies the result
// back (deterministic; a test transport, not a fast one).
struct hht_group {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<std::vector<uint8_t>> slot;

    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

#ifndef HHT_SINK_SLOTS
#define HHT_SINK_SLOTS 2
#endif
#ifndef HHT_SINK_CUT_DIV
#define HHT_SINK_CUT_DIV 8            // leaf sink: the final range's last 1/DIV becomes a range of its own (0: no cut)
#endif
constexpr uint32_t kSinkCutDiv = HHT_SINK_CUT_DIV;
constexpr int kSinkSlots = HHT_SINK_SLOTS;   // leaf-sink staging buffers (row conversion -> host copy)
#ifndef HHT_UNITS_PER_WARP
#define HHT_UNITS_PER_WARP 8
#endif
constexpr uint64_t kUnitsPerWarp = HHT_UNITS_PER_WARP;   // fused tail: split parents below this many per warp
#ifndef HHT_TAIL_SPLIT_PER_WARP
#define HHT_TAIL_SPLIT_PER_WARP 1     // many parents: the last (this many x warps) parents are split ...
#endif
#ifndef HHT_TAIL_SPLIT_K
#define HHT_TAIL_SPLIT_K 32           // ... into units of this many chunks (0: no split)
#endif
constexpr uint64_t kTailSplitPerWarp = HHT_TAIL_SPLIT_PER_WARP;
constexpr uint32_t kTailSplitK = HHT_TAIL_SPLIT_K;
constexpr int kFusedThreadsHost = 512;                     // k_fused block size (hht_kernels.cu kFusedThreads)

struct hht_ctx {
    hht_opts opts{};
    int sms = 148;
    cudaStream_t st = nullptr;
    cudaStream_t own_st = nullptr;              // the ctx's own stream (st may be a borrowed one)
    cudaStream_t cst2 = nullptr;                // W > 1: the fused tail's grid allreduce, overlapped
    cudaEvent_t ev_tail = nullptr, ev_ar = nullptr;
    Buf dense2[2];                              // W > 1: leaf grids of two consecutive ranges
    int dense_slot = 0;
    struct Deferred {                           // a fused-tail range whose grid allreduce is in flight
        bool pending = false;
        int l = 0;
        uint32_t r0 = 0, r1 = 0, n = 0;
        bool all_children = false;
        uint32_t* grids = nullptr;
    } deferred;
    bool own_comm = true;                       // false: comm is the caller's (opts.nccl_comm)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, tb0 = nullptr, tb1 = nullptr, ee0 = nullptr, ee1 = nullptr;
    ncclComm_t comm = nullptr;
    hht_group* group = nullptr;        // borrowed (opts.group)
    std::string err;
    size_t budget = 0;
    int grid[4][2] = {};
    int tail_grid[2] = {};
    int tail16_grid[2] = {};
    int fused_grid[2] = {};
    int split_grid = 0;             // resident k_split blocks (persistent tile loop)
    bool pref_pass = true, pref_tail = true;   // opts.prefetch (0 = auto)
    int pf_pass = 1;                           // list passes: 0 descriptor only, 1 registers, 2 bulk-copy ring
    bool circle = false;                       // opts.variant is a circumcircle test (1 or 2)
    int circle_var = 0;                        // opts.variant: 1 lattice units, 2 (m, b) units
    int grid_circle[3][2] = {};

    // last call
    int N = 0, D = 0, B = 0, H = 0, ntrees = 0;
    uint64_t T = 0;
    bool int64 = false;
    bool have = false;
    std::vector<uint8_t> tree_half;         // HHT_ALPHA / HHT_BETA per tree
    std::vector<int64_t> tree_E;            // global points per tree

    Buf stage_in, packed, errflag, beta, stats, tiles, tilectr, totals, rng, bounds, vtmp, dense, gv, leafrows, units;
    Buf fusedctr;                    // k_fused work counter (u32) + rastered-pair counter (u64)
    Buf img, edgeB, edgetiles;       // edge front end: staged image, BETA points, look-back words
    Buf small;                       // latency path scratch (k_small)
    Buf small_g;                     // latency path lists / frontiers when they exceed shared memory
    bool edges_valid = false;        // x->packed holds the last hht_detect_image's edge points
    std::vector<uint64_t> tree_pt_off;   // last detect: tree t's points in x->packed (local)
    std::vector<uint32_t> tree_pt_n;
    bool lines_ok = false;               // removal post-pass cached for the last detect
    std::vector<hht_leaf> lines_host;
    std::vector<int64_t> lines_img;      // [B+1] row offsets per image
    std::vector<std::pair<uint64_t, uint32_t>> lines_sup;   // (line index, point index in its tree)
    bool lines_sup_sorted = false;
    int rm_grid[2] = {0, 0};             // co-resident k_rm blocks (cooperative launch)
    int mid_grid[2] = {0, 0};            // co-resident k_mid blocks (cooperative launch)
    int64_t edge_na = 0, edge_nb = 0;
    // leaf sink (hht_set_leaf_sink): double-buffered row staging, copied on its own stream
    void* sink = nullptr;                // hht_leaf rows, or packed 8-byte rows (sink_packed)
    bool sink_packed = false;
    int64_t sink_cap = 0;
    uint64_t sink_n = 0;
    cudaStream_t cst = nullptr;
    Buf sinkrows[kSinkSlots];
    Buf treeoff;                         // hht_result_tree_offsets
    cudaEvent_t ev_conv[kSinkSlots] = {}, ev_copy[kSinkSlots] = {};
    bool copy_pending[kSinkSlots] = {};
    int sink_slot = 0;
    // pinned host memory that kernels write directly (mapped, UVA): small per-split readbacks
    Totals* totals_h = nullptr;
    RangeInfo* range_h = nullptr;
    uint64_t* misc_h = nullptr;
    bool errflag_dirty = true;              // errflag may be non-zero (see detect_impl)
    uint64_t alloc_gen = 0;                 // Buf generations
    struct H2dCache {                       // h2d_cached: the bytes a buffer last received
        const Buf* b = nullptr;
        uint64_t gen = 0;
        std::vector<uint8_t> bytes;
    } cache_small, cache_beta;
    uint32_t* fin_h = nullptr;              // the one-launch paths' mapped host block (kFinish* layout)
    uint32_t* fin_m = nullptr;
    uint8_t* pin = nullptr;                 // pinned staging for small host<->device copies of one call
    size_t pin_used = 0;
    Totals* totals_m = nullptr;      // device-side pointers of the same memory
    RangeInfo* range_m = nullptr;
    uint64_t* misc_m = nullptr;
    std::vector<Level> lv;
    Grow rec[64];
    Grow leaves;
    std::vector<Record> rec_host[64];
    bool rec_host_ok[64] = {};
    std::vector<LeafRec> leaves_host;
    bool leaves_host_ok = false;
    hht_stats stat{};
    hht_profile prof{};
    std::vector<ProfEv> pev;
    size_t pev_used = 0;
    std::vector<hht_launch> launch_log;
};

namespace {


// Levels covered by the dense tail: lists exist down to level D - tail_depth. 6: the fused tail
// streams level D-6 lists and rasters the 16x16 leaf grids of the level-(D-4) grandchildren (no
// level D-5 lists); 5 (auto when D >= 5): 16x16 leaf grids of level D-4, rastered straight from
// level D-5 lists by the fused tail; 4: 16x16 grids from level D-4 lists; 3: 8x8 grids from level
// D-3 lists.
int tail_depth(const hht_ctx* x) {
    const int want = x->opts.tail_depth ? (int)x->opts.tail_depth : 5;
    if (want >= 6 && x->D >= 6 && !x->circle) return 6;
    if (want >= 5 && x->D >= 5) return 5;
    return (want >= 4 && x->D >= 4) ? 4 : 3;
}

// With the fused tail and D >= 6, the last list pass (parent level D-6) skips the count-ahead: the
// fused tail rasters all children of the level-(D-5) regions and takes their votes from the grids.
bool no_count_ahead(const hht_ctx* x) { return !x->circle && tail_depth(x) == 5 && x->D >= 6; }

// The fused tail ends the list levels (tail_depth 5 or 6): the leaf sink's final cut applies there.
bool fused_tail(const hht_ctx* x) { return !x->circle && x->D >= 6 && tail_depth(x) >= 5; }

hht_status set_err(hht_ctx* x, hht_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (x) x->err = buf;
    return s;
}

#define CK(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return set_err(x, HHT_ECUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_),   \
                           __FILE__, __LINE__, #expr);                                            \
    } while (0)

#define CKN(expr)                                                                                 \
    do {                                                                                          \
        ncclResult_t r_ = (expr);                                                                 \
        if (r_ != ncclSuccess)                                                                    \
            return set_err(x, HHT_ENCCL, "NCCL error %s at %s:%d (%s)", ncclGetErrorString(r_),   \
                           __FILE__, __LINE__, #expr);                                            \
    } while (0)

#define TRY(expr)                                                                                 \
    do {                                                                                          \
        hht_status s_ = (expr);                                                                   \
        if (s_ != HHT_OK) return s_;                                                              \
    } while (0)

// Ensure capacity (contents are NOT preserved). exact: allocate exactly `bytes` (list buffers,
// which are accounted against the budget); otherwise grow geometrically.
hht_status ensure(hht_ctx* x, Buf& b, size_t bytes, bool exact = false) {
    if (bytes <= b.cap) return HHT_OK;
    size_t want = exact ? bytes : std::max(bytes, b.cap + b.cap / 2);
    want = (want + 255) & ~size_t(255);
    if (b.p) CK(cudaFreeAsync(b.p, x->st));
    b.p = nullptr;
    b.cap = 0;
    cudaError_t e = cudaMallocAsync(&b.p, want, x->st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(x, HHT_ENOMEM, "device allocation of %zu bytes failed (%s)", want, cudaGetErrorString(e));
    }
    b.cap = want;
    b.gen = ++x->alloc_gen;
    return HHT_OK;
}

hht_status release(hht_ctx* x, Buf& b) {
    if (b.p) CK(cudaFreeAsync(b.p, x->st));
    b.p = nullptr;
    b.cap = 0;
    return HHT_OK;
}

// Ensure capacity, preserving the first `keep` bytes.
hht_status grow(hht_ctx* x, Grow& g, size_t elem, uint64_t need) {
    if (need * elem <= g.b.cap) return HHT_OK;
    size_t want = std::max<size_t>(need * elem, g.b.cap * 2);
    want = (want + 255) & ~size_t(255);
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, want, x->st);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(x, HHT_ENOMEM, "device allocation of %zu bytes failed (%s)", want, cudaGetErrorString(e));
    }
    if (g.n) CK(cudaMemcpyAsync(p, g.b.p, g.n * elem, cudaMemcpyDeviceToDevice, x->st));
    if (g.b.p) CK(cudaFreeAsync(g.b.p, x->st));
    g.b.p = p;
    g.b.cap = want;
    return HHT_OK;
}

// Profiling: event pair around one launch.
int prof_begin(hht_ctx* x, int cls, uint64_t bytes) {
    if (!x->opts.profile) return -1;
    if (x->pev_used == x->pev.size()) {
        ProfEv e{};
        if (cudaEventCreate(&e.a) != cudaSuccess || cudaEventCreate(&e.b) != cudaSuccess) return -1;
        x->pev.push_back(e);
    }
    ProfEv& e = x->pev[x->pev_used];
    e.cls = cls;
    e.bytes = bytes;
    e.ops = 0;
    cudaEventRecord(e.a, x->st);
    return (int)x->pev_used++;
}
void prof_end(hht_ctx* x, int id) {
    if (id >= 0) cudaEventRecord(x->pev[id].b, x->st);
}

bool multi(const hht_ctx* x) { return x->comm != nullptr || x->group != nullptr; }

enum CollType { C_U32, C_U64, C_I64 };
enum CollOp { C_SUM, C_MIN, C_MAX };

template <class T>
void host_reduce(T* acc, const T* v, size_t n, CollOp op) {
    for (size_t i = 0; i < n; ++i)
        acc[i] = op == C_SUM ? (T)(acc[i] + v[i]) : op == C_MIN ? std::min(acc[i], v[i]) : std::max(acc[i], v[i]);
}

// Allreduce of `count` elements from device `send` into device `recv` (may alias), over NCCL or the
// in-process group. Asynchronous on the ctx stream for NCCL; synchronous for the group.
hht_status coll_allreduce(hht_ctx* x, const void* send, void* recv, size_t count, CollType t, CollOp op,
                          cudaStream_t stream = nullptr) {
    if (!multi(x) || count == 0) return HHT_OK;
    const cudaStream_t sm = stream ? stream : x->st;
    if (x->comm) {
        const ncclDataType_t dt = t == C_U32 ? ncclUint32 : t == C_U64 ? ncclUint64 : ncclInt64;
        const ncclRedOp_t ro = op == C_SUM ? ncclSum : op == C_MIN ? ncclMin : ncclMax;
        CKN(ncclAllReduce(send, recv, count, dt, ro, x->comm, sm));
        return HHT_OK;
    }
    hht_group* g = x->group;
    const size_t es = t == C_U32 ? 4 : 8, bytes = count * es;
    const int r = x->opts.rank;
    g->slot[r].resize(bytes);
    CK(cudaMemcpyAsync(g->slot[r].data(), send, bytes, cudaMemcpyDeviceToHost, sm));
    CK(cudaStreamSynchronize(sm));
    g->barrier();                                  // every rank's contribution is staged
    std::vector<uint8_t> acc(g->slot[0]);
    for (int k = 1; k < g->world; ++k) {
        if (g->slot[k].size() != bytes) return set_err(x, HHT_EMISMATCH, "group allreduce sizes differ");
        if (t == C_U32) host_reduce((uint32_t*)acc.data(), (const uint32_t*)g->slot[k].data(), count, op);
        else if (t == C_U64) host_reduce((uint64_t*)acc.data(), (const uint64_t*)g->slot[k].data(), count, op);
        else host_reduce((int64_t*)acc.data(), (const int64_t*)g->slot[k].data(), count, op);
    }
    g->barrier();                                  // every rank has read every slot
    CK(cudaMemcpyAsync(recv, acc.data(), bytes, cudaMemcpyHostToDevice, sm));
    CK(cudaStreamSynchronize(sm));
    return HHT_OK;
}

hht_status allreduce_sum_u32(hht_ctx* x, uint32_t* buf, size_t count) {
    if (!multi(x) || count == 0) return HHT_OK;
    const int id = prof_begin(x, 7, count * 4);
    TRY(coll_allreduce(x, buf, buf, count, C_U32, C_SUM));
    prof_end(x, id);
    return HHT_OK;
}

hht_status sync(hht_ctx* x) {
    CK(cudaStreamSynchronize(x->st));
    return HHT_OK;
}

// Read a value a kernel wrote into mapped pinned host memory (after a stream synchronisation).
template <class T>
T read_mapped(const T* p) {
    std::atomic_thread_fence(std::memory_order_acquire);
    T t;
    memcpy(&t, (const void*)p, sizeof t);
    return t;
}

// Small copies of one call go through the ctx's pinned staging area (async DMA; a pageable copy costs
// a host bounce and ~10 us each); the area is reused from the start by the next call, which is safe
// because every call synchronises its stream before returning.
constexpr size_t kPinBytes = 256 * 1024;
void* pin_take(hht_ctx* x, size_t bytes) {
    const size_t off = (x->pin_used + 15) & ~(size_t)15;
    if (!x->pin || off + bytes > kPinBytes) return nullptr;
    x->pin_used = off + bytes;
    return x->pin + off;
}
hht_status h2d_small(hht_ctx* x, void* dst, const void* src, size_t bytes) {
    void* p = pin_take(x, bytes);
    if (p) {
        memcpy(p, src, bytes);
        src = p;
    }
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, x->st));
    return HHT_OK;
}

// Host-to-device copy of a small constant block into `b`, skipped when `b` (same allocation) already
// holds exactly these bytes from an earlier call: repeated same-shape calls on the latency path then
// issue no copy at all. Every other write of `b` must drop the cache (c.b = nullptr).
hht_status h2d_cached(hht_ctx* x, hht_ctx::H2dCache& c, Buf& b, const void* src, size_t bytes) {
    if (c.b == &b && c.gen == b.gen && c.bytes.size() == bytes && memcmp(c.bytes.data(), src, bytes) == 0)
        return HHT_OK;
    TRY(h2d_small(x, b.p, src, bytes));
    c.b = &b;
    c.gen = b.gen;
    c.bytes.assign((const uint8_t*)src, (const uint8_t*)src + bytes);
    return HHT_OK;
}

size_t sink_row_bytes(const hht_ctx* x) { return x->sink_packed ? sizeof(uint64_t) : sizeof(hht_leaf); }

// Leaf sink: rows of leaves [first, first + n) -> host, overlapped with the traversal.
hht_status stream_leaves(hht_ctx* x, uint64_t first, uint64_t n) {
    if (!x->sink || n == 0 || x->sink_n >= (uint64_t)x->sink_cap) return HHT_OK;
    const uint64_t k = std::min<uint64_t>(n, (uint64_t)x->sink_cap - x->sink_n);
    const size_t rb = sink_row_bytes(x);
    const int s = x->sink_slot;
    x->sink_slot = (s + 1) % kSinkSlots;
    Buf& b = x->sinkrows[s];
    if (b.cap < k * rb) {
        if (x->copy_pending[s]) CK(cudaEventSynchronize(x->ev_copy[s]));   // before freeing its buffer
        x->copy_pending[s] = false;
        TRY(ensure(x, b, k * rb));
    }
    if (x->copy_pending[s]) CK(cudaStreamWaitEvent(x->st, x->ev_copy[s], 0));   // buffer reuse
    if (x->sink_packed)
        CK(launch_leaf_packed((const LeafRec*)x->leaves.b.p + first, k, (uint64_t*)b.p, x->st));
    else
        CK(launch_leaf_rows((const LeafRec*)x->leaves.b.p + first, k, (const uint8_t*)x->beta.p, x->H,
                            (uint32_t*)b.p, x->st));
    CK(cudaEventRecord(x->ev_conv[s], x->st));
    CK(cudaStreamWaitEvent(x->cst, x->ev_conv[s], 0));
    CK(cudaMemcpyAsync((uint8_t*)x->sink + x->sink_n * rb, b.p, k * rb, cudaMemcpyDefault, x->cst));
    CK(cudaEventRecord(x->ev_copy[s], x->cst));
    x->copy_pending[s] = true;
    x->sink_n += k;
    return HHT_OK;
}

// ---------------------------------------------------------------------------------------------
// split: threshold the votes of the children of parents P[r0, r0+Fp) into level child_level.
// ---------------------------------------------------------------------------------------------
hht_status do_split(hht_ctx* x, int child_level, Level& P, uint32_t r0, uint32_t Fp, const uint32_t* V,
                    const uint32_t* VL, bool derive_ne = false) {
    if (Fp == 0) return HHT_OK;
    Level& C = x->lv[child_level];
    const bool leaf = child_level == x->D;
    // lists are read by write passes (levels < D-TK) and the dense tail (level D-TK); for D = 2 the
    // count-only pass reads the roots' lists (the points themselves)
    const bool need_lists = child_level <= x->D - (x->circle ? 2 : tail_depth(x));
    const uint64_t nch = 4ull * Fp;
    if (!leaf) {
        TRY(ensure(x, C.tree, nch * 4));
        TRY(ensure(x, C.a, nch * 4));
        TRY(ensure(x, C.c, nch * 4));
        TRY(ensure(x, C.parent, nch * 4));
        TRY(ensure(x, C.len, nch * 4));
        TRY(ensure(x, C.votes_g, nch * 4));
        TRY(ensure(x, C.off, (nch + 1) * 8));
        TRY(ensure(x, C.choff, (nch + 1) * 8));
        TRY(ensure(x, C.nf, nch * 4));
        if (need_lists) TRY(ensure(x, C.nfoff, nch * 8));
    } else {
        TRY(grow(x, x->leaves, sizeof(LeafRec), x->leaves.n + nch));
    }
    const bool record = x->opts.record_levels != 0;
    if (record) TRY(grow(x, x->rec[child_level], sizeof(Record), x->rec[child_level].n + nch));
    const uint32_t ntiles = (Fp + kSplitThreads - 1) / kSplitThreads;
    TRY(ensure(x, x->tiles, (size_t)(ntiles + kScanBlocks) * sizeof(TileDesc)));
    CK(cudaMemsetAsync(x->tiles.p, 0, (size_t)ntiles * sizeof(TileDesc), x->st));
    CK(cudaMemsetAsync(x->tilectr.p, 0, 4, x->st));

    SplitArgs a{};
    a.V = V;
    a.VL = VL;
    a.Fp = Fp;
    a.p_tree = (const uint32_t*)P.tree.p + r0;
    a.p_a = (const uint32_t*)P.a.p + r0;
    a.p_c = (const uint32_t*)P.c.p + r0;
    a.parent_base = r0;
    a.derive_ne = derive_ne;
    a.p_votes = derive_ne ? (const uint32_t*)P.votes_g.p + r0 : nullptr;
    a.p_len = derive_ne ? (const uint32_t*)P.len.p + r0 : nullptr;
    a.child_level = child_level;
    a.leaf_level = leaf;
    a.need_lists = need_lists;
    // offsets are read by chunk maps and range selection: list levels, and level D-1 when a
    // count-only pass runs there (circle variants, depth < 3; the tails never read them). The child ->
    // next-index map is read by the passes over the parents' lists (list levels) and that count-only
    // pass; a leaf grid's gathers need neither.
    const bool count_only = x->circle || x->D < 3;
    a.write_off = need_lists || (child_level == x->D - 1 && count_only);
    a.record = record;
    a.T = x->T;
    // the pass over the deepest list level (a write pass, a fused tail rastering only split children,
    // or the count-only pass) reads its children's map: levels up to one below the deepest lists
    const int list_max = x->D - (count_only ? 2 : tail_depth(x));
    a.nf = child_level <= list_max + 1 ? (uint32_t*)C.nf.p : nullptr;
    a.nfoff = need_lists ? (uint64_t*)C.nfoff.p : nullptr;
    a.out = C.frontier();
    a.rec = record ? (Record*)x->rec[child_level].b.p + x->rec[child_level].n : nullptr;
    a.leaves = leaf ? (LeafRec*)x->leaves.b.p + x->leaves.n : nullptr;
    a.tiles = (TileDesc*)x->tiles.p;
    a.scan_seg = (TileDesc*)x->tiles.p + ntiles;
    a.tile_counter = (uint32_t*)x->tilectr.p;
    a.stats = (unsigned long long*)x->stats.p;
    a.totals = x->totals_m;
    a.ntiles = ntiles;
    const uint64_t bytes = (uint64_t)Fp * (16 + (VL != V ? 16 : 0) + 12 + (leaf ? 0 : 16) + (record ? 64 : 0));
    const int id = prof_begin(x, 4, bytes);
    CK(launch_split(a, x->split_grid, x->st));
    prof_end(x, id);
    TRY(sync(x));
    const Totals t = read_mapped(x->totals_h);
    if (record) x->rec[child_level].n += nch;
    if (leaf) {
        const uint64_t first = x->leaves.n;
        x->leaves.n += t.F;
        return stream_leaves(x, first, t.F);
    }
    C.F = (uint32_t)t.F;
    C.S = t.S;
    C.C = t.C;
    if (x->opts.profile) x->prof.bytes[4] += (uint64_t)C.F * 36;
    if (need_lists && C.F) {
        TRY(ensure(x, C.chunks, std::max<uint64_t>(C.C, 1) * sizeof(ChunkDesc)));
        const int id2 = prof_begin(x, 5, C.C * sizeof(ChunkDesc) + (uint64_t)C.F * 36);
        CK(launch_chunk_map((const uint64_t*)C.choff.p, (const uint64_t*)C.off.p, (const uint32_t*)C.len.p,
                            (const uint32_t*)C.a.p, (const uint32_t*)C.c.p, (const uint32_t*)C.tree.p,
                            (const uint8_t*)x->beta.p, C.F, (ChunkDesc*)C.chunks.p, x->st));
        prof_end(x, id2);
    }
    return HHT_OK;
}

PassArgs pass_args(hht_ctx* x, Level& P, int level) {
    PassArgs a{};
    a.list = P.list;
    a.list_base = P.list_base;
    a.chunks = (const ChunkDesc*)P.chunks.p;
    a.chunk_bounds = (const uint64_t*)x->bounds.p;
    a.level = level;
    a.D = x->D;
    a.N = x->N;
    a.one = 1;
    // 16x16 raster fixed point (Raster16): 2^fx_s >= 32 * 3N > G_SW - 1 of any line crossing a
    // level-(D-4) region; fx_m = ceil(2^(24+fx_s) / 3N) < 2^30 + 1, fx_mlo = floor(...)
    {
        const uint64_t n3 = 3ull * (uint64_t)x->N;
        int s = 0;
        while ((1ull << s) < 32 * n3) ++s;
        a.fx_s = (uint32_t)s;
        a.fx_m = (uint32_t)(((1ull << (24 + s)) + n3 - 1) / n3);
        a.fx_mlo = (uint32_t)((1ull << (24 + s)) / n3);
    }
    return a;
}

hht_status run_pass(hht_ctx* x, int mode, const PassArgs& a, uint64_t pairs, uint64_t written) {
    const int cls = mode == MODE_COUNT ? 1 : ((mode == MODE_WRITE || mode == MODE_WRITE_NC) ? 2 : 3);
    const int id = prof_begin(x, cls, pairs * 4 + written * 4);
    const int grid = x->circle ? x->grid_circle[mode][x->int64 ? 1 : 0] : x->grid[mode][x->int64 ? 1 : 0];
    CK(launch_pass(mode, x->int64, x->circle ? 1 : x->pf_pass, x->circle_var, a, grid, x->st));
    prof_end(x, id);
    x->stat.pairs += pairs;
    return HHT_OK;
}

// Choose [q0, q1) over the level-lc frontier; W > 1 agrees on the smallest proposal. The frontier
// holds the split children of parents R_(lc-1)[r0, r1). When those parents are the whole parent
// frontier, everything fits and one rank runs, the range is the whole level and its bounds are
// known on the host (no kernel, no synchronisation); the chunk range then covers all parents.
hht_status choose_range(hht_ctx* x, int lc, uint32_t q0, uint64_t cap_entries, bool all, RangeInfo* out,
                        uint32_t r0, uint32_t r1) {
    Level& C = x->lv[lc];
    Level& P = x->lv[lc - 1];
    if (!multi(x) && q0 == 0 && r0 == 0 && r1 == P.F && (all || C.S <= cap_entries)) {
        *out = RangeInfo{C.F, 0, C.S, 0, P.C, P.S};
        CK(launch_set_bounds((uint64_t*)x->bounds.p, 0, P.C, x->st));
        return HHT_OK;
    }
    const int id = prof_begin(x, 6, 0);
    CK(launch_range((const uint64_t*)C.off.p, (const uint32_t*)C.parent.p, C.F, q0, cap_entries,
                    all ? C.F : 0, (const uint64_t*)P.off.p, (const uint64_t*)P.choff.p,
                    (const uint32_t*)P.len.p, lc == 1, (RangeInfo*)x->rng.p, (uint64_t*)x->bounds.p, x->range_m,
                    x->st));
    prof_end(x, id);
    if (multi(x) && !all) {
        // min over ranks of the proposed end, then recompute with the agreed end
        TRY(coll_allreduce(x, (const char*)x->rng.p + offsetof(RangeInfo, q1), x->vtmp.p, 1, C_U64, C_MIN));
        CK(launch_copy_u32((uint32_t*)x->misc_m, (const uint32_t*)x->vtmp.p, 2, x->st));
        TRY(sync(x));
        const uint64_t q1 = read_mapped(x->misc_h);
        CK(launch_range((const uint64_t*)C.off.p, (const uint32_t*)C.parent.p, C.F, q0, cap_entries, q1,
                        (const uint64_t*)P.off.p, (const uint64_t*)P.choff.p, (const uint32_t*)P.len.p,
                        lc == 1, (RangeInfo*)x->rng.p, (uint64_t*)x->bounds.p, x->range_m, x->st));
    }
    TRY(sync(x));
    *out = read_mapped(x->range_h);
    return HHT_OK;
}

// Dense tail at level L = D-TK (D >= 3): lv[L] holds the lists of R_L[r0, r1) and lv[L+1] holds
// R_(L+1) (its split children, without lists). One pass counts the 2^TK x 2^TK leaf grid of every
// R_L region; every deeper level is then split from votes gathered out of the grids (a region's
// votes = the sum of its diagonal leaves), down to the leaves.
hht_status gather_levels(hht_ctx* x, int L, int c0, uint32_t anc_base, Level& Own, int TK,
                         const uint32_t* owner_parent = nullptr, const uint32_t* grids = nullptr);

hht_status tail(hht_ctx* x, int L, uint32_t r0, uint32_t r1) {
    const int TK = x->D - L;
    const uint32_t cells = 1u << (2 * TK);
    Level& P = x->lv[L];
    const uint32_t n = r1 - r0;
    if (n == 0) return HHT_OK;
    TRY(ensure(x, x->dense, (size_t)n * cells * 4));
    CK(cudaMemsetAsync(x->dense.p, 0, (size_t)n * cells * 4, x->st));
    CK(launch_bounds((const uint64_t*)P.off.p, (const uint64_t*)P.choff.p, (const uint32_t*)P.len.p, r0, r1, L == 0,
                     (RangeInfo*)x->rng.p, (uint64_t*)x->bounds.p, x->range_m, x->st));
    PassArgs a = pass_args(x, P, L);
    a.nf_rbase = r0;
    a.votes = (uint32_t*)x->dense.p;
    const int id = prof_begin(x, 3, 0);
    if (TK == 4) CK(launch_tail16(x->int64, x->pref_tail, a, x->tail16_grid[x->int64 ? 1 : 0], x->st));
    else CK(launch_tail(x->int64, a, x->tail_grid[x->int64 ? 1 : 0], x->st));
    prof_end(x, id);
    TRY(sync(x));
    const uint64_t pairs = read_mapped(x->range_h).pairs;
    if (id >= 0) {
        x->pev[id].bytes = pairs * 4 + (uint64_t)n * cells * 4;
        // raster step = 8 instructions per (line, leaf column): advance the height, extract the
        // drop, form the table address, load the column mask, two counter adds, two state updates
        x->pev[id].ops = pairs * (1ull << TK) * 8;
    }
    x->stat.pairs += pairs;
    TRY(allreduce_sum_u32(x, (uint32_t*)x->dense.p, (size_t)n * cells));
    return gather_levels(x, L, L + 2, r0, P, TK);
}

// Levels c0 .. D from the leaf grids of the grid owners R_L[anc_base, ...): parents R_(c-1), a
// child's votes = the sum of its diagonal leaves, then the split of level c.
hht_status gather_levels(hht_ctx* x, int L, int c0, uint32_t anc_base, Level& Own, int TK,
                         const uint32_t* owner_parent, const uint32_t* grids) {
    if (!grids) grids = (const uint32_t*)x->dense.p;
    for (int c = c0; c <= x->D; ++c) {
        Level& Pc = x->lv[c - 1];
        if (Pc.F == 0) return HHT_OK;
        const int hops = c - 1 - L;
        GatherChain chain{};
        for (int h = 0; h < hops; ++h) chain.parent[h] = (const uint32_t*)x->lv[c - 1 - h].parent.p;
        TRY(ensure(x, x->gv, 16ull * Pc.F));
        const int g = prof_begin(x, 5, (16ull + 8 + 4ull * hops + 16ull * (1u << (x->D - c))) * Pc.F);
        CK(launch_gather(grids, anc_base, (const uint32_t*)Own.a.p, (const uint32_t*)Own.c.p,
                         (const uint32_t*)Pc.a.p, (const uint32_t*)Pc.c.p, chain, hops, TK, x->D - c, Pc.F,
                         (uint32_t*)x->gv.p, owner_parent, x->st));
        prof_end(x, g);
        TRY(do_split(x, c, Pc, 0, Pc.F, (const uint32_t*)x->gv.p, (const uint32_t*)x->gv.p));
    }
    return HHT_OK;
}

// Fused tail at parent level l = D-5: lv[l] holds the lists of R_l[r0, r1). One k_fused pass rasters
// 16x16 leaf grids straight from those lists: of the split children R_(l+1) (their votes came from
// the previous pass's count-ahead), or, when `all_children` (that pass ran without count-ahead),
// of all 4 children of each parent, whose votes are then the grids' diagonal sums and whose split
// happens here. Levels l+2 .. D are split from the grids.
// With `gp` (tail_depth 6), R_l has no lists: each work unit r streams the list of its parent in
// gp = lv[l-1] (all_children only).
// The grid work of a fused-tail range with all children rastered: votes of the level-L children as
// diagonal sums, their split, then levels L+1 .. D from the grids.
hht_status tail_grid_levels(hht_ctx* x, int l, uint32_t r0, uint32_t r1, uint32_t n, const uint32_t* grids) {
    const int L = l + 1;
    Level& P = x->lv[l];
    TRY(ensure(x, x->gv, 16ull * (r1 - r0)));
    const int g = prof_begin(x, 5, (uint64_t)n * 64 + 16ull * (r1 - r0));
    CK(launch_grid_diag(grids, r1 - r0, (uint32_t*)x->gv.p, x->st));
    prof_end(x, g);
    TRY(do_split(x, L, P, r0, r1 - r0, (const uint32_t*)x->gv.p, (const uint32_t*)x->gv.p));
    return gather_levels(x, L, L + 1, r0, x->lv[L], 4, (const uint32_t*)x->lv[L].parent.p, grids);
}

// W > 1: the previous range's leaf grids were summed over the ranks on a second stream while this
// rank went on with the next range (its list pass and fused tail); finish that range now.
hht_status flush_deferred(hht_ctx* x) {
    if (!x->deferred.pending) return HHT_OK;
    x->deferred.pending = false;
    CK(cudaStreamWaitEvent(x->st, x->ev_ar, 0));
    const auto d = x->deferred;
    return tail_grid_levels(x, d.l, d.r0, d.r1, d.n, d.grids);
}

hht_status tail_fused(hht_ctx* x, int l, uint32_t r0, uint32_t r1, bool all_children, Level* gp = nullptr) {
    const int L = l + 1;
    Level& P = x->lv[l];
    Level& C = x->lv[L];
    if (r1 == r0) return HHT_OK;
    const uint32_t n = all_children ? 4 * (r1 - r0) : C.F;
    if (n == 0) return HHT_OK;
    // W > 1 with all children rastered: the grid allreduce overlaps the next range (double-buffered
    // grids, flush_deferred); else it is on the critical path
    const bool defer = multi(x) && all_children && !gp;
    Buf& gb = defer ? x->dense2[x->dense_slot] : x->dense;
    TRY(ensure(x, gb, (size_t)n * kTail16Cells * 4));
    uint32_t* grids = (uint32_t*)gb.p;
    CK(cudaMemsetAsync(grids, 0, (size_t)n * kTail16Cells * 4, x->st));
    TRY(ensure(x, x->fusedctr, 256));
    CK(cudaMemsetAsync(x->fusedctr.p, 0, 24, x->st));
    // streamed pairs: host-known when the parents are the whole level, else from the device
    const bool host_pairs = !gp && r0 == 0 && r1 == P.F;
    if (!host_pairs && !gp)
        CK(launch_bounds((const uint64_t*)P.off.p, (const uint64_t*)P.choff.p, (const uint32_t*)P.len.p, r0, r1,
                         l == 0, (RangeInfo*)x->rng.p, (uint64_t*)x->bounds.p, x->range_m, x->st));
    PassArgs a = pass_args(x, gp ? *gp : P, l);
    a.nf = all_children ? nullptr : (const uint32_t*)C.nf.p;
    a.nf_rbase = r0;
    a.q0 = 0;
    a.q1 = all_children ? n : C.F;
    a.votes = grids;
    a.p_choff = (const uint64_t*)(gp ? gp->choff.p : P.choff.p);
    if (gp) {
        a.gp_parent = (const uint32_t*)P.parent.p;
        a.gp_a = (const uint32_t*)P.a.p;
        a.gp_c = (const uint32_t*)P.c.p;
    }
    a.r_lo = r0;
    a.r_hi = r1;
    a.work = (uint32_t*)x->fusedctr.p;
    a.child_pairs = (unsigned long long*)((char*)x->fusedctr.p + 8);
    a.all_children = all_children ? 1u : 0u;
    // few parents for the warps (C3, small ranges): split each parent's chunks into work units so that
    // every warp gets work until the end (a unit's partial raster batches are its only extra cost)
    const uint64_t nwarps = (uint64_t)x->fused_grid[x->int64 ? 1 : 0] * (kFusedThreadsHost / 32);
    if (!gp && x->opts.tail_units != 2 && x->opts.tail_units != 3 && (uint64_t)(r1 - r0) < kUnitsPerWarp * nwarps) {
        const uint64_t target = kUnitsPerWarp * nwarps;
        const uint64_t cap = target + (r1 - r0) + 1;        // sum of ceil(chunks_r / K) <= chunks / K + parents
        TRY(ensure(x, x->units, cap * 8 + 16));
        uint32_t* nk = (uint32_t*)((char*)x->units.p + cap * 8);
        CK(launch_units(a.p_choff, r0, r1, (uint32_t)target, r0, 0, (uint2*)x->units.p, nk, x->st));
        a.units = (const uint2*)x->units.p;
        a.nunits = nk;
        a.unit_k = nk + 1;
    } else if (!gp && x->opts.tail_units != 2 && kTailSplitK > 0 && kTailSplitPerWarp > 0) {
        // (tail_units 3 takes this path whatever the parent count: tests)
        // many parents: whole parents first, then the last ones in pieces of kTailSplitK chunks (the
        // end of the launch otherwise waits for the warps that took the last large parents)
        const uint64_t ns = std::min<uint64_t>(r1 - r0, kTailSplitPerWarp * nwarps);
        const uint32_t r_split = r1 - (uint32_t)ns;
        // sum over the split parents of ceil(chunks_r / K) <= their chunks / K + ns <= P.C / K + ns
        const uint64_t cap = (r_split - r0) + ns + P.C / kTailSplitK + 1;
        TRY(ensure(x, x->units, cap * 8 + 16));
        uint32_t* nk = (uint32_t*)((char*)x->units.p + cap * 8);
        CK(launch_units(a.p_choff, r0, r1, 0, r_split, kTailSplitK, (uint2*)x->units.p, nk, x->st));
        a.units = (const uint2*)x->units.p;
        a.nunits = nk;
        a.unit_k = nk + 1;
    }
    const int id = prof_begin(x, 3, 0);
    CK(launch_fused(x->int64, a, x->fused_grid[x->int64 ? 1 : 0], x->st));
    prof_end(x, id);
    uint64_t pairs = P.S, child_pairs = 0;
    if (!host_pairs || id >= 0) {      // the device counters are read only when needed
        CK(launch_copy_u32((uint32_t*)x->misc_m, (const uint32_t*)((char*)x->fusedctr.p + 8), 4, x->st));
        TRY(sync(x));
        if (gp) pairs = read_mapped(x->misc_h + 1);
        else if (!host_pairs) pairs = read_mapped(x->range_h).pairs;
        child_pairs = read_mapped(x->misc_h);
    }
    if (id >= 0) {
        x->pev[id].bytes = pairs * 4 + (uint64_t)n * kTail16Cells * 4;
        // raster steps: 16 leaf columns x 8 instructions per (line, child) pair (see tail()), plus the
        // 4 exact child tests (subtract + compare) per parent entry
        x->pev[id].ops = child_pairs * 16 * 8 + pairs * 4 * 2;
    }
    x->stat.pairs += pairs;
    if (defer) {
        TRY(flush_deferred(x));                       // the previous range, in range order
        CK(cudaEventRecord(x->ev_tail, x->st));
        CK(cudaStreamWaitEvent(x->cst2, x->ev_tail, 0));
        TRY(coll_allreduce(x, grids, grids, (size_t)n * kTail16Cells, C_U32, C_SUM, x->cst2));
        CK(cudaEventRecord(x->ev_ar, x->cst2));
        x->deferred.pending = true;
        x->deferred.l = l;
        x->deferred.r0 = r0;
        x->deferred.r1 = r1;
        x->deferred.n = n;
        x->deferred.all_children = true;
        x->deferred.grids = grids;
        x->dense_slot ^= 1;
        return HHT_OK;
    }
    TRY(allreduce_sum_u32(x, grids, (size_t)n * kTail16Cells));
    if (!all_children) return gather_levels(x, L, L + 1, 0, C, 4);
    return tail_grid_levels(x, l, r0, r1, n, grids);
}

// tail_depth 6 at l = D-6: lv[l] holds the lists of a parent range and lv[l+1] its split children
// R_(l+1) (votes from the last count-ahead, no lists). The fused tail streams each child's parent
// list and rasters the leaf grids of all 4 children of the child; R_(l+1) is processed in pieces
// whose grids (4 KB per region) stay within a quarter of the list budget (at most 1 GiB).
hht_status tail_grandparent(hht_ctx* x, int l) {
    Level& C = x->lv[l + 1];
    const uint32_t F = C.F;
    const uint64_t per = 4ull * kTail16Cells * 4;
    const uint64_t capn = std::max<uint64_t>(1, std::min<uint64_t>(x->budget / 4, 1ull << 30) / per);
    for (uint32_t q0 = 0; q0 < F;) {
        const uint32_t q1 = (uint32_t)std::min<uint64_t>(F, q0 + capn);
        TRY(tail_fused(x, l + 1, q0, q1, true, &x->lv[l]));
        q0 = q1;
    }
    return HHT_OK;
}

// Preconditions: lv[l] holds the lists of R_l[r0, r1) and lv[l+1] holds R_(l+1) = the split
// children of R_l[r0, r1) with NF_(l+1). Processes everything below.
hht_status descend(hht_ctx* x, int l, uint32_t r0, uint32_t r1) {
    const int lc = l + 1;
    if (lc >= x->D) return HHT_OK;
    if (!x->circle && x->D >= 3 && l == x->D - tail_depth(x)) {
        if (tail_depth(x) == 6) return tail_grandparent(x, l);
        return tail_depth(x) == 5 ? tail_fused(x, l, r0, r1, no_count_ahead(x)) : tail(x, l, r0, r1);
    }
    Level& P = x->lv[l];
    Level& C = x->lv[lc];
    const uint32_t Fc = C.F;
    if (Fc == 0) return HHT_OK;

    if (lc == x->D - 1) {
        // count-only pass: level-D votes of the children of R_(D-1), then the leaves.
        RangeInfo ri{};
        TRY(choose_range(x, lc, 0, 0, true, &ri, r0, r1));
        TRY(ensure(x, C.votes, 16ull * Fc));
        CK(cudaMemsetAsync(C.votes.p, 0, 16ull * Fc, x->st));
        PassArgs a = pass_args(x, P, l);
        a.nf = (const uint32_t*)C.nf.p;
        a.nf_rbase = r0;
        a.q0 = 0;
        a.q1 = Fc;
        a.votes = (uint32_t*)C.votes.p;
        TRY(run_pass(x, MODE_COUNT2, a, ri.pairs, 0));
        TRY(allreduce_sum_u32(x, (uint32_t*)C.votes.p, 4ull * Fc));
        return do_split(x, x->D, C, 0, Fc, (const uint32_t*)C.votes.p, (const uint32_t*)C.votes.p, !x->circle);
    }

    uint32_t q0 = 0;
    bool final_cut = false;          // the last range has been cut once already (leaf sink, below)
    while (q0 < Fc) {
        // list budget left for this level: everything not held by the active ancestor levels.
        // Buffer capacities persist across ranges and calls (steady state allocates nothing);
        // idle deeper buffers are released only under budget pressure.
        size_t active = 0;
        for (int k = 1; k < lc; ++k) active += x->lv[k].list_own.cap;
        const size_t avail = x->budget > active ? x->budget - active : 0;
        const uint64_t cap = (lc == x->D - 2 ? avail : avail / 3) / 4;
        RangeInfo ri{};
        TRY(choose_range(x, lc, q0, cap, false, &ri, r0, r1));
        // With a leaf sink, the leaves of the last range are copied to the host after all compute: when
        // the detection's final piece at the last list level would be large, cut its last eighth into
        // a range of its own, so that the copy of the rest overlaps that eighth's tail. (Halving the
        // final piece repeatedly, 1/2, 1/4, ..., measured worse on C5: +1.5, +4.5, +8.7 ms e2e with 1, 3
        // and 5 cuts, since a small piece leaves most warps of its fused tail idle.)
        if (kSinkCutDiv > 0 && x->sink && !final_cut && ri.q1 == Fc && q0 > 0 && r1 == P.F && fused_tail(x) &&
            lc == x->D - tail_depth(x) && Fc - q0 >= 64) {
            final_cut = true;
            const uint32_t qf = q0 + (Fc - q0) - (Fc - q0) / kSinkCutDiv;
            CK(launch_range((const uint64_t*)C.off.p, (const uint32_t*)C.parent.p, C.F, q0, cap, qf,
                            (const uint64_t*)P.off.p, (const uint64_t*)P.choff.p, (const uint32_t*)P.len.p,
                            lc == 1, (RangeInfo*)x->rng.p, (uint64_t*)x->bounds.p, x->range_m, x->st));
            TRY(sync(x));
            ri = read_mapped(x->range_h);
        }
        const uint32_t q1 = (uint32_t)ri.q1;
        const uint64_t entries = ri.s_hi - ri.s_lo;
        if (entries * 4 > avail)
            return set_err(x, HHT_ENOMEM, "level %d region list of %llu entries exceeds the list budget (%zu B free)",
                           lc, (unsigned long long)entries, avail);
        if (entries * 4 + 64 > C.list_own.cap) {
            size_t deeper = 0;
            for (int k = lc + 1; k < (int)x->lv.size(); ++k) deeper += x->lv[k].list_own.cap;
            if (active + entries * 4 + deeper > x->budget)
                for (int k = lc + 1; k < (int)x->lv.size(); ++k) TRY(release(x, x->lv[k].list_own));
            TRY(release(x, C.list_own));
            TRY(ensure(x, C.list_own, std::max<uint64_t>(entries, 1) * 4 + 64, true));   // + bulk-copy slack
        }
        C.list = (const uint32_t*)C.list_own.p;
        C.list_base = ri.s_lo;
        const uint32_t nq = q1 - q0;
        TRY(ensure(x, C.cursor, 4ull * nq));
        TRY(ensure(x, C.votes, 16ull * nq));
        CK(cudaMemsetAsync(C.cursor.p, 0, 4ull * nq, x->st));
        CK(cudaMemsetAsync(C.votes.p, 0, 16ull * nq, x->st));
        PassArgs a = pass_args(x, P, l);
        a.nf = (const uint32_t*)C.nf.p;
        a.nf_rbase = r0;
        a.q0 = q0;
        a.q1 = q1;
        a.nfoff = (const uint64_t*)C.nfoff.p;
        a.c_list_base = ri.s_lo;
        a.c_cursor = (uint32_t*)C.cursor.p;
        a.c_list = (uint32_t*)C.list_own.p;
        a.votes = (uint32_t*)C.votes.p;
        const bool nc = no_count_ahead(x) && lc == x->D - 5;
        TRY(run_pass(x, nc ? MODE_WRITE_NC : MODE_WRITE, a, ri.pairs, entries));
        x->stat.ranges += 1;
        if (nc) {                     // level lc+1 votes come from the fused tail's grids
            TRY(descend(x, lc, q0, q1));
            q0 = q1;
            continue;
        }
        const uint32_t* VL = (const uint32_t*)C.votes.p;
        if (multi(x)) {
            TRY(ensure(x, C.votes_local, 16ull * nq));
            CK(cudaMemcpyAsync(C.votes_local.p, C.votes.p, 16ull * nq, cudaMemcpyDeviceToDevice, x->st));
            VL = (const uint32_t*)C.votes_local.p;
            TRY(allreduce_sum_u32(x, (uint32_t*)C.votes.p, 4ull * nq));
        }
        TRY(do_split(x, lc + 1, C, q0, nq, (const uint32_t*)C.votes.p, VL, !x->circle));
        TRY(descend(x, lc, q0, q1));
        q0 = q1;
    }
    // W > 1: a deferred fused-tail range reads this level's frontier (lv[lc]), which the caller's next
    // range rebuilds: finish it before returning
    return flush_deferred(x);
}

hht_status check_args(hht_ctx* x, const int32_t* points, int64_t n_total, int32_t N, int32_t D, int64_t T) {
    if (!x) return HHT_EINVAL;
    if (n_total < 0) return set_err(x, HHT_EINVAL, "n < 0");
    if (n_total > 0 && !points) return set_err(x, HHT_EINVAL, "points is NULL");
    if (((uintptr_t)points & 7) != 0) return set_err(x, HHT_EINVAL, "points must be 8-byte aligned");
    if (N < 1 || N > 65536) return set_err(x, HHT_EINVAL, "N must be in [1, 65536] (16-bit packed coordinates)");
    if (D < 1 || D > 30) return set_err(x, HHT_EINVAL, "depth must be in [1, 30]");
    if (x->sink && x->sink_packed && D > 16)
        return set_err(x, HHT_EINVAL, "a packed leaf sink needs depth <= 16 (16-bit i, j)");
    if (T < 1) return set_err(x, HHT_EINVAL, "threshold must be >= 1");
    if (x->opts.halves == 0 || (x->opts.halves & ~3u)) return set_err(x, HHT_EINVAL, "bad halves");
    // |G| < 5 N 2^D must fit the signed width
    const long double mag = 5.0L * (long double)N * (long double)(1ull << D);
    if (mag >= 4.6e18L) return set_err(x, HHT_EOVERFLOW, "5*N*2^depth >= 2^62: exact int64 arithmetic impossible");
    if (n_total > 0xFFFFFFFFll) return set_err(x, HHT_EINVAL, "more than 2^32-1 points per rank");
    if (x->opts.variant > HHT_FHT_CIRCLE_MB) return set_err(x, HHT_EINVAL, "unknown variant");
    // circle test: the squared radius 2 s^2 (4 ex^2 + 9 N^2) of a child of the root must fit 63 bits
    if (x->opts.variant == HHT_FHT_CIRCLE && 13.0L * N * (long double)N * powl(2.0L, 2.0L * D - 1) >= 9.2e18L)
        return set_err(x, HHT_EOVERFLOW, "13 N^2 2^(2 depth - 1) >= 2^63: circle radius overflows 64 bits");
    // (m, b)-unit circle: (1 + N^2)(4 + 9 N^2) s^2 for a child of the root (s = 2^(D-1)) in 126 bits
    if (x->opts.variant == HHT_FHT_CIRCLE_MB &&
        (1.0L + (long double)N * N) * (4.0L + 9.0L * N * (long double)N) * powl(2.0L, 2.0L * D - 2) >= powl(2.0L, 126))
        return set_err(x, HHT_EOVERFLOW, "(1 + N^2)(4 + 9 N^2) 4^(depth-1) >= 2^126: (m, b) circle radius overflows");
    return HHT_OK;
}

// Latency path: eligible when every per-level array of the traversal fits one block's shared memory
// (lists: a line crosses at most 2^(l+1) - 1 regions of level l, so a level-l list holds at most
// sum_t n_t (2^(l+1) - 1) entries; frontier: a split region holds > T entries), one rank, the exact
// test, and opts.latency_path != 2. One k_small launch does every level; one synchronisation reads
// the per-level record counts, the leaf count and the statistics.
void small_bounds(const hht_ctx* x, uint64_t& S, uint64_t& F) {
    uint64_t n = 0;
    for (int t = 0; t < x->ntrees; ++t) n += x->tree_pt_n[t];
    S = std::max<uint64_t>(n * ((1ull << x->D) - 1), 1);   // list levels 0 .. D-1
    F = S / (x->T + 1) + x->ntrees + 1;
}

// 0: multi-kernel path; 1: latency path with shared-memory scratch; 2: latency path with the two
// candidate lists in device (L2-resident) memory and the frontier arrays in shared memory, for lists
// up to kSmallGlobalMaxS entries (profiles/r01_latency.md)
hht_status finish_small(hht_ctx* x, int id, uint32_t path);

// 3: the mid-size latency path (k_mid, hht_mid.cu): one cooperative launch over the GPU, lists and
// frontier in device memory, for lists up to kMidMaxS entries (opts.latency_path 3 forces it when the
// bounds admit it).
int small_mode(const hht_ctx* x) {
    if (x->opts.latency_path == 2 || multi(x) || x->circle || x->D > 24 || x->ntrees > 4096) return 0;
    uint64_t S, F;
    small_bounds(x, S, F);
    if (S >= (1ull << 32)) return 0;
    const uint32_t Fc = (uint32_t)std::min<uint64_t>(F, S + 1);
    const bool mid_ok = S <= kMidMaxS && (uint64_t)Fc + 1 <= (uint64_t)kMidMaxTiles * kMidThreads;
    if (x->opts.latency_path == 3) return mid_ok ? 3 : 0;
    if (small_smem_bytes((uint32_t)S, Fc) <= kSmallSmemMax) return 1;
    if (S <= kSmallGlobalMaxS && small_frontier_bytes(Fc) <= kSmallSmemMax) return 2;
    return mid_ok ? 3 : 0;
}

hht_status detect_mid(hht_ctx* x, const int32_t* dev_pts, uint64_t npts) {
    const int D = x->D;
    const uint32_t nt = (uint32_t)x->ntrees;
    uint64_t n = 0;
    for (uint32_t t = 0; t < nt; ++t) n += x->tree_pt_n[t];
    uint64_t Smax, Fmax;
    small_bounds(x, Smax, Fmax);
    Fmax = std::min<uint64_t>(Fmax, Smax + 1) + 1;
    const uint64_t tiles = (Fmax + kMidThreads - 1) / kMidThreads;
    // host-written block: tree offsets and counts, per-level counts, control words, record pointers
    const uint64_t words = 3ull * nt + (D + 2) + 8 + 2ull * (D + 1) + 16;
    TRY(ensure(x, x->small, words * 4));
    uint32_t* w = (uint32_t*)x->small.p;
    MidArgs a{};
    uint64_t* d_off = (uint64_t*)w; w += 2ull * nt;
    uint32_t* d_n = w; w += nt;
    a.counts = w; w += D + 2;
    a.ctl = w; w += 8;
    w = (uint32_t*)(((uintptr_t)w + 7) & ~(uintptr_t)7);
    Record** d_rec = (Record**)w;
    std::vector<Record*> h_rec(D + 1);
    for (int l = 0; l <= D; ++l) {
        const uint64_t cap = l == 0 ? nt : 4 * Fmax;
        TRY(grow(x, x->rec[l], sizeof(Record), cap));
        h_rec[l] = (Record*)x->rec[l].b.p;
    }
    TRY(grow(x, x->leaves, sizeof(LeafRec), 4 * Fmax));
    // device scratch: 2 lists (Smax) + 2 x 6 frontier arrays (Fmax + 1) + 2 x cv (4 Fmax) + cursor,
    // loff, lcoff (4 Fmax) + app (Fmax) + tiles (3 tiles)
    const uint64_t F1 = Fmax + 1;
    const uint64_t Cmax = Smax / kChunk + Fmax + 1;       // chunks of one level: sum ceil(len / 256)
    auto up4 = [](uint64_t w) { return (w + 3) & ~3ull; };   // every array 16-byte aligned (vector access)
    const uint64_t swords = 2 * (8 * F1 + up4(4 * Fmax)) + 2 * up4(Smax) + 2 * up4(Cmax) + 3 * up4(4 * Fmax) +
                            up4(Fmax) + up4(3 * tiles) + 64;
    TRY(ensure(x, x->small_g, swords * 4));
    uint32_t* g = (uint32_t*)x->small_g.p;               // 256-byte aligned
    for (int b = 0; b < 2; ++b) {
        a.fd[b] = (uint4*)g; g += 8 * F1;
        a.cv[b] = g; g += up4(4 * Fmax);
    }
    a.list[0] = g; g += up4(Smax);
    a.list[1] = g; g += up4(Smax);
    for (int b = 0; b < 2; ++b) {
        a.chunkmap[b] = g; g += up4(Cmax);
    }
    a.cursor = g; g += up4(4 * Fmax);
    a.loff = g; g += up4(4 * Fmax);
    a.lcoff = g; g += up4(4 * Fmax);
    a.app = g; g += up4(Fmax);
    a.tiles = g;
    {
        std::vector<uint32_t> h(words, 0);
        memcpy(h.data(), x->tree_pt_off.data(), 8ull * nt);
        memcpy(h.data() + 2ull * nt, x->tree_pt_n.data(), 4ull * nt);
        memcpy((char*)h.data() + ((char*)d_rec - (char*)x->small.p), h_rec.data(), sizeof(Record*) * (D + 1));
        // counts: zeroed by k_mid; ctl[3] (range flag): 0 on upload, re-armed by k_mid
        TRY(h2d_cached(x, x->cache_small, x->small, h.data(), words * 4));
    }
    a.packed = (uint32_t*)x->packed.p;
    a.pts = (const int2*)dev_pts;          // staged and range-checked by k_mid itself
    a.npts = dev_pts ? npts : 0;
    a.fin = x->fin_m;
    a.tree_off = d_off;
    a.tree_n = d_n;
    a.tree_beta = (const uint8_t*)x->beta.p;
    a.ntrees = nt;
    a.N = x->N;
    a.D = D;
    a.T = x->T;
    a.record = x->opts.record_levels ? 1u : 0u;
    a.rec = d_rec;
    a.leaves = (LeafRec*)x->leaves.b.p;
    a.stats = (unsigned long long*)x->stats.p;
    if (!x->mid_grid[x->int64 ? 1 : 0]) x->mid_grid[x->int64 ? 1 : 0] = x->sms * mid_blocks_per_sm(x->int64);
    const int id = prof_begin(x, 1, n * 4 * (uint64_t)(D + 1));
    CK(launch_mid(a, x->int64, x->mid_grid[x->int64 ? 1 : 0], x->st));
    prof_end(x, id);
    return finish_small(x, id, 2);
}

hht_status detect_small(hht_ctx* x, const int32_t* dev_pts, uint64_t npts) {
    const int D = x->D;
    const uint32_t nt = (uint32_t)x->ntrees;
    uint64_t n = 0;
    for (uint32_t t = 0; t < nt; ++t) n += x->tree_pt_n[t];
    uint64_t Smax, Fmax;
    small_bounds(x, Smax, Fmax);
    Fmax = std::min<uint64_t>(Fmax, Smax + 1);
    // global scratch: tree offsets and counts, per-level counts, record pointers
    const uint64_t words = 3ull * nt + (D + 2) + 2ull * (D + 1) + 16;
    TRY(ensure(x, x->small, words * 4));
    uint32_t* w = (uint32_t*)x->small.p;
    SmallArgs a{};
    a.smem_S = (uint32_t)((Smax + 3) & ~3ull);    // list stride, a multiple of 4 (small_smem_bytes)
    a.smem_F = (uint32_t)Fmax;
    uint64_t* d_off = (uint64_t*)w; w += 2ull * nt;
    uint32_t* d_n = w; w += nt;
    a.counts = w; w += D + 2;
    w = (uint32_t*)(((uintptr_t)w + 7) & ~(uintptr_t)7);
    Record** d_rec = (Record**)w;
    std::vector<Record*> h_rec(D + 1);
    for (int l = 0; l <= D; ++l) {
        const uint64_t cap = l == 0 ? nt : 4 * Fmax;
        TRY(grow(x, x->rec[l], sizeof(Record), cap));
        h_rec[l] = (Record*)x->rec[l].b.p;
    }
    TRY(grow(x, x->leaves, sizeof(LeafRec), 4 * Fmax));
    a.global_scratch = small_mode(x) == 2 ? 1u : 0u;
    if (a.global_scratch) {
        // the two candidate lists in one device buffer (the frontier arrays stay in shared memory)
        TRY(ensure(x, x->small_g, 8ull * a.smem_S));
        a.list[0] = (uint32_t*)x->small_g.p;
        a.list[1] = a.list[0] + a.smem_S;
    }
    {   // one host-to-device copy of everything the launch needs (offsets, counts, zeroed counters,
        // record pointers), laid out exactly as in `x->small`
        std::vector<uint32_t> h(words, 0);
        memcpy(h.data(), x->tree_pt_off.data(), 8ull * nt);
        memcpy(h.data() + 2ull * nt, x->tree_pt_n.data(), 4ull * nt);
        memcpy((char*)h.data() + ((char*)d_rec - (char*)x->small.p), h_rec.data(), sizeof(Record*) * (D + 1));
        TRY(h2d_cached(x, x->cache_small, x->small, h.data(), words * 4));   // k_small zeroes the counts
    }
    a.packed = (uint32_t*)x->packed.p;
    a.pts = (const int2*)dev_pts;          // staged and range-checked by k_small itself
    a.npts = dev_pts ? npts : 0;
    a.fin = x->fin_m;
    a.tree_off = d_off;
    a.tree_n = d_n;
    a.tree_beta = (const uint8_t*)x->beta.p;
    a.ntrees = nt;
    a.N = x->N;
    a.D = D;
    a.T = x->T;
    a.rec = d_rec;
    a.leaves = (LeafRec*)x->leaves.b.p;
    a.stats = (unsigned long long*)x->stats.p;
    const int id = prof_begin(x, 1, n * 4 * (uint64_t)(D + 1));
    CK(launch_small(a, x->int64, x->st));
    prof_end(x, id);
    return finish_small(x, id, 1);
}

// Results of a one-launch traversal (k_small, k_mid): per-level record counts, leaves and statistics
// in one synchronisation, with the range check of the staged points.
hht_status finish_small(hht_ctx* x, int id, uint32_t path) {
    const int D = x->D;
    CK(cudaEventRecord(x->ev1, x->st));
    TRY(sync(x));
    x->errflag_dirty = false;
    std::atomic_thread_fence(std::memory_order_acquire);
    const uint32_t* counts = x->fin_h + 1;
    const uint64_t* st = (const uint64_t*)(x->fin_h + kFinishStatsWord);
    if (x->fin_h[0]) return set_err(x, HHT_ERANGE, "a point lies outside [0, N)^2");
    for (int l = 0; l <= D; ++l) x->rec[l].n = x->opts.record_levels ? counts[l] : 0;
    x->leaves.n = counts[D + 1];
    x->stat.tests = st[kStatTests];
    x->stat.votes = st[kStatVotes];
    x->stat.leaves = st[kStatLeaves];
    for (int l = 0; l <= D && l < 64; ++l) {
        x->stat.visited[l] = st[kStatVisited0 + l];
        x->stat.split[l] = st[kStatSplit0 + l];
    }
    x->stat.latency_path = path;
    TRY(stream_leaves(x, 0, x->leaves.n));
    if (x->sink) {
        CK(cudaStreamSynchronize(x->cst));
        x->stat.leaves_streamed = x->sink_n;
        x->stat.d2h_bytes += x->sink_n * sink_row_bytes(x);
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, x->ev0, x->ev1));
    x->stat.ms = ms;
    x->launch_log.clear();
    if (x->opts.profile && id >= 0) {
        float m = 0;
        if (cudaEventElapsedTime(&m, x->pev[id].a, x->pev[id].b) == cudaSuccess) {
            x->prof.ms[1] += m;
            x->prof.launches[1] += 1;
            x->prof.bytes[1] += x->pev[id].bytes;
            x->launch_log.push_back({1u, 0, x->pev[id].bytes, (double)m});
        }
    }
    x->have = true;
    return HHT_OK;
}

hht_status detect_impl(hht_ctx* x, const int32_t* points, const int64_t* offsets, int32_t B, int32_t N,
                       int32_t D, int64_t T, const int64_t* tree_offsets = nullptr, bool prepacked = false) {
    x->pin_used = 0;                  // the previous call synchronised: its staging is free
    x->deferred.pending = false;      // a failed previous call may have left one
    // offsets: per image [B+1] (every point enters each of the image's trees); tree_offsets: per
    // tree [B*H+1] (tree t = image t/H, halves in ALPHA, BETA order; each point in one tree)
    if (!x) return HHT_EINVAL;
    x->err.clear();
    x->have = false;
    const int Hh = (x->opts.halves & HHT_ALPHA ? 1 : 0) + (x->opts.halves & HHT_BETA ? 1 : 0);
    const int64_t* segs = tree_offsets ? tree_offsets : offsets;
    const int nseg = tree_offsets ? B * Hh : B;
    if (B < 1 || !segs) return set_err(x, HHT_EINVAL, "need B >= 1 images and host offsets");
    if (segs[0] != 0) return set_err(x, HHT_EINVAL, "offsets[0] must be 0");
    for (int b = 0; b < nseg; ++b)
        if (segs[b + 1] < segs[b]) return set_err(x, HHT_EINVAL, "offsets must be non-decreasing");
    const int64_t n = segs[nseg];
    TRY(check_args(x, points, n, N, D, T));

    x->N = N;
    x->D = D;
    x->T = (uint64_t)T;
    x->B = B;
    x->H = (x->opts.halves & HHT_ALPHA ? 1 : 0) + (x->opts.halves & HHT_BETA ? 1 : 0);
    x->ntrees = B * x->H;
    // |G| < 5 N 2^D (exact test); the circle test also squares 2 G(centre): |L2| < 10 N 2^D
    x->int64 = x->opts.force_int64 || !((x->circle ? 10.0L : 5.0L) * N * (long double)(1ull << D) < 2147483647.0L);
    memset(&x->stat, 0, sizeof x->stat);
    memset(&x->prof, 0, sizeof x->prof);
    x->pev_used = 0;
    x->stat.levels = D + 1;
    x->stat.int_bits = x->int64 ? 64 : 32;
    x->stat.images = B;
    for (int l = 0; l < 64; ++l) {
        x->rec[l].n = 0;
        x->rec_host_ok[l] = false;
    }
    x->leaves.n = 0;
    x->leaves_host_ok = false;
    x->sink_n = 0;
    x->sink_slot = 0;        // same staging-slot sequence every call: buffers sized once, then reused
    if ((int)x->lv.size() < D + 1) x->lv.resize(D + 1);
    for (auto& L : x->lv) {
        L.F = 0;
        L.S = L.C = 0;
        L.list = nullptr;
    }

    CK(cudaSetDevice(x->opts.device));
    CK(cudaEventRecord(x->ev0, x->st));

    // trees and per-tree point counts (global over ranks)
    x->tree_half.assign(x->ntrees, 0);
    std::vector<int64_t> local_n(nseg);
    for (int b = 0; b < nseg; ++b) local_n[b] = segs[b + 1] - segs[b];
    {
        int t = 0;
        for (int b = 0; b < B; ++b)
            for (uint32_t h : {HHT_ALPHA, HHT_BETA})
                if (x->opts.halves & h) x->tree_half[t++] = (uint8_t)h;
    }
    std::vector<int64_t> global_n = local_n;
    if (multi(x)) {
        // argument agreement: min and max of (N, D, T, halves, B, per-tree mode) must coincide
        int64_t prm[6] = {N, D, T, (int64_t)x->opts.halves, B, tree_offsets ? 1 : 0};
        TRY(ensure(x, x->vtmp, std::max<size_t>(8 * 12, 8 * (size_t)nseg)));
        CK(cudaMemcpyAsync(x->vtmp.p, prm, sizeof prm, cudaMemcpyHostToDevice, x->st));
        CK(cudaMemcpyAsync((char*)x->vtmp.p + 48, prm, sizeof prm, cudaMemcpyHostToDevice, x->st));
        TRY(coll_allreduce(x, x->vtmp.p, x->vtmp.p, 6, C_I64, C_MIN));
        TRY(coll_allreduce(x, (char*)x->vtmp.p + 48, (char*)x->vtmp.p + 48, 6, C_I64, C_MAX));
        int64_t got[12];
        CK(cudaMemcpyAsync(got, x->vtmp.p, sizeof got, cudaMemcpyDeviceToHost, x->st));
        TRY(sync(x));
        for (int i = 0; i < 6; ++i)
            if (got[i] != got[6 + i]) return set_err(x, HHT_EMISMATCH, "ranks disagree on (N, depth, threshold, halves, images)");
        CK(cudaMemcpyAsync(x->vtmp.p, local_n.data(), 8 * (size_t)nseg, cudaMemcpyHostToDevice, x->st));
        TRY(coll_allreduce(x, x->vtmp.p, x->vtmp.p, nseg, C_I64, C_SUM));
        CK(cudaMemcpyAsync(global_n.data(), x->vtmp.p, 8 * (size_t)nseg, cudaMemcpyDeviceToHost, x->st));
        TRY(sync(x));
    }
    x->tree_E.assign(x->ntrees, 0);
    for (int t = 0; t < x->ntrees; ++t) x->tree_E[t] = global_n[tree_offsets ? t : t / x->H];
    x->tree_pt_off.assign(x->ntrees, 0);
    x->tree_pt_n.assign(x->ntrees, 0);
    for (int t = 0; t < x->ntrees; ++t) {
        const int sgi = tree_offsets ? t : t / x->H;
        x->tree_pt_off[t] = (uint64_t)segs[sgi];
        x->tree_pt_n[t] = (uint32_t)local_n[sgi];
    }
    x->lines_ok = false;

    // K0: stage + validate (reject before any traversal; collective over ranks)
    if (!prepacked) x->edges_valid = false;
    if (prepacked) {
        if (x->packed.cap < (size_t)n * 4) return set_err(x, HHT_EINVAL, "internal: prepacked points exceed the buffer");
    } else {
        TRY(ensure(x, x->packed, std::max<int64_t>(n, 1) * 4 + 64));   // + bulk-copy slack
    }
    // the one-launch paths (k_small, k_mid) stage and range-check the points themselves (no k_stage
    // launch, no errflag)
    const int smode = small_mode(x);
    const bool stage_in_small = smode != 0;
    // errflag is 0 on entry: zeroed at create, re-armed after the multi-kernel path's range check; a
    // call that failed in between leaves it dirty
    if (!stage_in_small) {
        if (x->errflag_dirty) CK(cudaMemsetAsync(x->errflag.p, 0, 4, x->st));
        x->errflag_dirty = true;
    }
    const int32_t* small_pts = nullptr;
    if (n > 0 && !prepacked) {   // prepacked: x->packed already holds in-range points (edge front end)
        const int32_t* dev_pts = points;
        cudaPointerAttributes pa{};
        cudaError_t e = cudaPointerGetAttributes(&pa, points);
        if (e != cudaSuccess) cudaGetLastError();
        const bool on_device = e == cudaSuccess && (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged);
        if (!on_device) {
            TRY(ensure(x, x->stage_in, (size_t)n * 8));
            CK(cudaMemcpyAsync(x->stage_in.p, points, (size_t)n * 8, cudaMemcpyHostToDevice, x->st));
            x->stat.h2d_bytes += (uint64_t)n * 8;
            dev_pts = (const int32_t*)x->stage_in.p;
        }
        if (stage_in_small) {
            small_pts = dev_pts;
        } else {
            const int id = prof_begin(x, 0, (uint64_t)n * 12);
            CK(launch_stage(dev_pts, (uint64_t)n, N, (uint32_t*)x->packed.p, (uint32_t*)x->errflag.p, x->st));
            prof_end(x, id);
        }
    }
    if (smode) {
        // latency path: no synchronisation before the traversal; the range check is read with the
        // results (an out-of-range point still fails the call with HHT_ERANGE, nothing is returned);
        // the kernels zero the statistics themselves
        std::vector<uint8_t> beta(x->ntrees);
        for (int t = 0; t < x->ntrees; ++t) beta[t] = x->tree_half[t] == HHT_BETA;
        TRY(ensure(x, x->beta, x->ntrees));
        TRY(h2d_cached(x, x->cache_beta, x->beta, beta.data(), x->ntrees));
        return smode == 3 ? detect_mid(x, small_pts, (uint64_t)n) : detect_small(x, small_pts, (uint64_t)n);
    }
    TRY(coll_allreduce(x, x->errflag.p, x->errflag.p, 1, C_U32, C_MAX));
    CK(launch_copy_u32((uint32_t*)x->misc_m, (const uint32_t*)x->errflag.p, 1, x->st));
    CK(cudaMemsetAsync(x->errflag.p, 0, 4, x->st));        // re-armed for the next call
    TRY(sync(x));
    x->errflag_dirty = false;
    if ((uint32_t)read_mapped(x->misc_h)) return set_err(x, HHT_ERANGE, "a point lies outside [0, N)^2");

    // stats accumulators
    CK(cudaMemsetAsync(x->stats.p, 0, kStatCount * 8, x->st));
    std::vector<uint8_t> beta(x->ntrees);
    for (int t = 0; t < x->ntrees; ++t) beta[t] = x->tree_half[t] == HHT_BETA;
    TRY(ensure(x, x->beta, x->ntrees));
    TRY(h2d_cached(x, x->cache_beta, x->beta, beta.data(), x->ntrees));

    // level 0: every tree's root ("each line ... passes through this region")
    uint64_t root_votes = 0, root_tests = 0, root_split = 0;
    std::vector<Record> r0rec;
    std::vector<uint32_t> h_tree, h_zero, h_len, h_votes;
    std::vector<uint64_t> h_off, h_choff;
    uint64_t chunks = 0, pairs0 = 0;
    for (int t = 0; t < x->ntrees; ++t) {
        const int b = t / x->H;
        const uint64_t E = (uint64_t)x->tree_E[t];
        r0rec.push_back({(uint32_t)t, 0, 0, (uint32_t)E});
        root_votes += E;
        root_tests += E;
        if (E > x->T) {                 // R6: the uniform split rule also applies at the root
            root_split++;
            root_tests += 4 * E;
            h_tree.push_back(t);
            h_zero.push_back(0);
            const uint64_t ln = (uint64_t)local_n[tree_offsets ? t : b];
            h_len.push_back((uint32_t)ln);
            h_votes.push_back((uint32_t)E);
            h_off.push_back((uint64_t)segs[tree_offsets ? t : b]);
            h_choff.push_back(chunks);
            chunks += (ln + kChunk - 1) / kChunk;
            pairs0 += ln;
        }
    }
    const uint32_t F0 = (uint32_t)h_tree.size();
    h_off.push_back((uint64_t)n);
    h_choff.push_back(chunks);
    x->stat.visited[0] = x->ntrees;
    x->stat.split[0] = root_split;
    if (x->opts.record_levels) {
        TRY(grow(x, x->rec[0], sizeof(Record), x->ntrees));
        CK(cudaMemcpyAsync(x->rec[0].b.p, r0rec.data(), r0rec.size() * sizeof(Record), cudaMemcpyHostToDevice, x->st));
        x->rec[0].n = x->ntrees;
    }
    Level& L0 = x->lv[0];
    L0.F = F0;
    L0.S = pairs0;
    L0.C = chunks;
    L0.list = (const uint32_t*)x->packed.p;
    L0.list_base = 0;
    if (F0 > 0) {
        TRY(ensure(x, L0.tree, F0 * 4ull));
        TRY(ensure(x, L0.a, F0 * 4ull));
        TRY(ensure(x, L0.c, F0 * 4ull));
        TRY(ensure(x, L0.parent, F0 * 4ull));
        TRY(ensure(x, L0.len, F0 * 4ull));
        TRY(ensure(x, L0.votes_g, F0 * 4ull));
        TRY(ensure(x, L0.off, (F0 + 1) * 8ull));
        TRY(ensure(x, L0.choff, (F0 + 1) * 8ull));
        TRY(ensure(x, L0.chunks, std::max<uint64_t>(chunks, 1) * sizeof(ChunkDesc)));
        CK(cudaMemcpyAsync(L0.tree.p, h_tree.data(), F0 * 4ull, cudaMemcpyHostToDevice, x->st));
        CK(cudaMemcpyAsync(L0.a.p, h_zero.data(), F0 * 4ull, cudaMemcpyHostToDevice, x->st));
        CK(cudaMemcpyAsync(L0.c.p, h_zero.data(), F0 * 4ull, cudaMemcpyHostToDevice, x->st));
        CK(cudaMemcpyAsync(L0.parent.p, h_tree.data(), F0 * 4ull, cudaMemcpyHostToDevice, x->st));
        CK(cudaMemcpyAsync(L0.len.p, h_len.data(), F0 * 4ull, cudaMemcpyHostToDevice, x->st));
        CK(cudaMemcpyAsync(L0.votes_g.p, h_votes.data(), F0 * 4ull, cudaMemcpyHostToDevice, x->st));
        CK(cudaMemcpyAsync(L0.off.p, h_off.data(), (F0 + 1) * 8ull, cudaMemcpyHostToDevice, x->st));
        CK(cudaMemcpyAsync(L0.choff.p, h_choff.data(), (F0 + 1) * 8ull, cudaMemcpyHostToDevice, x->st));
        CK(launch_chunk_map((const uint64_t*)L0.choff.p, (const uint64_t*)L0.off.p, (const uint32_t*)L0.len.p,
                            (const uint32_t*)L0.a.p, (const uint32_t*)L0.c.p, (const uint32_t*)L0.tree.p,
                            (const uint8_t*)x->beta.p, F0, (ChunkDesc*)L0.chunks.p, x->st));
        const uint64_t cb[2] = {0, chunks};
        CK(cudaMemcpyAsync(x->bounds.p, cb, sizeof cb, cudaMemcpyHostToDevice, x->st));
        TRY(ensure(x, L0.votes, 16ull * F0));
        CK(cudaMemsetAsync(L0.votes.p, 0, 16ull * F0, x->st));
        PassArgs a = pass_args(x, L0, 0);
        a.votes = (uint32_t*)L0.votes.p;
        a.nf_rbase = 0;
        TRY(run_pass(x, MODE_COUNT, a, pairs0, 0));
        const uint32_t* VL = (const uint32_t*)L0.votes.p;
        if (multi(x)) {
            TRY(ensure(x, L0.votes_local, 16ull * F0));
            CK(cudaMemcpyAsync(L0.votes_local.p, L0.votes.p, 16ull * F0, cudaMemcpyDeviceToDevice, x->st));
            VL = (const uint32_t*)L0.votes_local.p;
            TRY(allreduce_sum_u32(x, (uint32_t*)L0.votes.p, 4ull * F0));
        }
        TRY(do_split(x, 1, L0, 0, F0, (const uint32_t*)L0.votes.p, VL));
        TRY(descend(x, 0, 0, F0));
        TRY(flush_deferred(x));              // W > 1: the last range's grid work
    }

    // stats
    uint64_t st[kStatCount];
    CK(cudaMemcpyAsync(st, x->stats.p, sizeof st, cudaMemcpyDeviceToHost, x->st));
    CK(cudaEventRecord(x->ev1, x->st));
    TRY(sync(x));
    x->stat.tests = root_tests + st[kStatTests];
    x->stat.votes = root_votes + st[kStatVotes];
    x->stat.leaves = st[kStatLeaves];
    for (int l = 1; l <= D && l < 64; ++l) {
        x->stat.visited[l] = st[kStatVisited0 + l];
        x->stat.split[l] = st[kStatSplit0 + l];
    }
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, x->ev0, x->ev1));
    x->stat.ms = ms;
    if (x->sink) {
        CK(cudaStreamSynchronize(x->cst));
        for (int k = 0; k < kSinkSlots; ++k) x->copy_pending[k] = false;
        x->stat.leaves_streamed = x->sink_n;
        x->stat.d2h_bytes += x->sink_n * sink_row_bytes(x);
    }
    x->launch_log.clear();
    if (x->opts.profile) {
        for (size_t i = 0; i < x->pev_used; ++i) {
            float m = 0;
            if (cudaEventElapsedTime(&m, x->pev[i].a, x->pev[i].b) == cudaSuccess) {
                x->prof.ms[x->pev[i].cls] += m;
                x->prof.launches[x->pev[i].cls] += 1;
                x->prof.bytes[x->pev[i].cls] += x->pev[i].bytes;
                x->prof.ops[x->pev[i].cls] += x->pev[i].ops;
                x->launch_log.push_back({(uint32_t)x->pev[i].cls, 0, x->pev[i].bytes, (double)m});
            }
        }
    }
    x->have = true;
    return HHT_OK;
}

hht_status host_records(hht_ctx* x, int level) {
    if (x->rec_host_ok[level]) return HHT_OK;
    x->rec_host[level].resize(x->rec[level].n);
    if (x->rec[level].n)
        CK(cudaMemcpyAsync(x->rec_host[level].data(), x->rec[level].b.p, x->rec[level].n * sizeof(Record),
                           cudaMemcpyDeviceToHost, x->st));
    TRY(sync(x));
    x->rec_host_ok[level] = true;
    return HHT_OK;
}

hht_status host_leaves(hht_ctx* x) {
    if (x->leaves_host_ok) return HHT_OK;
    x->leaves_host.resize(x->leaves.n);
    if (x->leaves.n)
        CK(cudaMemcpyAsync(x->leaves_host.data(), x->leaves.b.p, x->leaves.n * sizeof(LeafRec),
                           cudaMemcpyDeviceToHost, x->st));
    TRY(sync(x));
    x->stat.d2h_bytes += x->leaves.n * sizeof(LeafRec);
    x->leaves_host_ok = true;
    return HHT_OK;
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

#ifndef HHT_BUILD_ID
#define HHT_BUILD_ID "unknown"
#endif
// "hht <version> sm_100a build <id>": id = sha256 of the sources, headers and nvcc flags (build.py
// build_id), the same for every build of the same kernels (bench.py matches ncu captures on it)
const char* hht_version(void) { return "hht 0.1.0 sm_100a build " HHT_BUILD_ID; }

const char* hht_status_str(hht_status s) {
    switch (s) {
        case HHT_OK: return "HHT_OK";
        case HHT_EINVAL: return "HHT_EINVAL";
        case HHT_ERANGE: return "HHT_ERANGE";
        case HHT_EOVERFLOW: return "HHT_EOVERFLOW";
        case HHT_ENOMEM: return "HHT_ENOMEM";
        case HHT_ECUDA: return "HHT_ECUDA";
        case HHT_ENCCL: return "HHT_ENCCL";
        case HHT_EMISMATCH: return "HHT_EMISMATCH";
        case HHT_ESTATE: return "HHT_ESTATE";
    }
    return "HHT_UNKNOWN";
}

hht_status hht_default_opts(hht_opts* o) {
    if (!o) return HHT_EINVAL;
    memset(o, 0, sizeof *o);
    o->device = 0;
    o->rank = 0;
    o->world = 1;
    o->halves = HHT_ALPHA | HHT_BETA;
    o->record_levels = 1;
    return HHT_OK;
}

hht_status hht_group_create(hht_group** out, int32_t world) {
    if (!out || world < 1) return HHT_EINVAL;
    hht_group* g = new (std::nothrow) hht_group();
    if (!g) return HHT_ENOMEM;
    g->world = world;
    g->slot.resize(world);
    *out = g;
    return HHT_OK;
}

void hht_group_destroy(hht_group* g) { delete g; }

hht_status hht_nccl_unique_id(void* out, size_t cap) {
    if (!out || cap < sizeof(ncclUniqueId)) return HHT_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return HHT_ENCCL;
    memcpy(out, &id, sizeof id);
    return HHT_OK;
}

hht_status hht_create(hht_ctx** out, const hht_opts* opts) {
    if (!out) return HHT_EINVAL;
    *out = nullptr;
    hht_opts o;
    if (opts) o = *opts; else hht_default_opts(&o);
    if (o.world < 1 || o.rank < 0 || o.rank >= o.world) return HHT_EINVAL;
    if (o.world > 1 && !o.nccl_id && !o.nccl_comm && !o.group) return HHT_EINVAL;
    if (o.group && (o.nccl_id || o.nccl_comm || o.group->world != o.world)) return HHT_EINVAL;
    if (o.halves == 0 || (o.halves & ~3u)) return HHT_EINVAL;
    if (!(o.tail_depth == 0 || (o.tail_depth >= 3 && o.tail_depth <= 6))) return HHT_EINVAL;
    hht_ctx* x = new (std::nothrow) hht_ctx();
    if (!x) return HHT_ENOMEM;
    x->opts = o;
    auto fail = [&](hht_status s) {
        hht_destroy(x);
        return s;
    };
    if (cudaSetDevice(o.device) != cudaSuccess) { cudaGetLastError(); return fail(HHT_ECUDA); }
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, o.device) != cudaSuccess) return fail(HHT_ECUDA);
    x->sms = prop.multiProcessorCount;
    if (cudaStreamCreateWithFlags(&x->own_st, cudaStreamNonBlocking) != cudaSuccess) return fail(HHT_ECUDA);
    x->st = o.stream ? (cudaStream_t)o.stream : x->own_st;
    if (cudaStreamCreateWithFlags(&x->cst, cudaStreamNonBlocking) != cudaSuccess) return fail(HHT_ECUDA);
    if (cudaStreamCreateWithFlags(&x->cst2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&x->ev_tail, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&x->ev_ar, cudaEventDisableTiming) != cudaSuccess)
        return fail(HHT_ECUDA);
    for (int k = 0; k < kSinkSlots; ++k)
        if (cudaEventCreateWithFlags(&x->ev_conv[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&x->ev_copy[k], cudaEventDisableTiming) != cudaSuccess)
            return fail(HHT_ECUDA);
    if (cudaEventCreate(&x->ev0) != cudaSuccess || cudaEventCreate(&x->ev1) != cudaSuccess ||
        cudaEventCreate(&x->tb0) != cudaSuccess || cudaEventCreate(&x->tb1) != cudaSuccess ||
        cudaEventCreate(&x->ee0) != cudaSuccess || cudaEventCreate(&x->ee1) != cudaSuccess)
        return fail(HHT_ECUDA);
    // keep freed pool memory cached across calls
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, o.device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    if (o.prefetch == 1) x->pref_pass = x->pref_tail = false;
    if (o.prefetch == 2) x->pref_pass = x->pref_tail = true;
    x->pf_pass = o.prefetch == 3 ? 2 : (x->pref_pass ? 1 : 0);
    for (int m = 0; m < 4; ++m)
        for (int w = 0; w < 2; ++w) x->grid[m][w] = x->sms * pass_blocks_per_sm(m, w == 1, x->pf_pass, 0);
    x->circle = o.variant == HHT_FHT_CIRCLE || o.variant == HHT_FHT_CIRCLE_MB;
    x->circle_var = x->circle ? (int)o.variant : 0;
    for (int m = 0; m < 3; ++m)
        for (int w = 0; w < 2; ++w)
            x->grid_circle[m][w] = x->sms * pass_blocks_per_sm(m, w == 1, 1, x->circle_var ? x->circle_var : 1);
    for (int w = 0; w < 2; ++w) x->tail_grid[w] = x->sms * tail_blocks_per_sm(w == 1);
    for (int w = 0; w < 2; ++w) x->tail16_grid[w] = x->sms * tail16_blocks_per_sm(w == 1, x->pref_tail);
    for (int w = 0; w < 2; ++w) x->fused_grid[w] = x->sms * fused_blocks_per_sm(w == 1);
    x->split_grid = x->sms * split_blocks_per_sm();
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return fail(HHT_ECUDA);
    x->budget = o.mem_budget ? o.mem_budget : (size_t)(0.70 * (double)fr);
    if (ensure(x, x->errflag, 256) || ensure(x, x->stats, kStatCount * 8) || ensure(x, x->tilectr, 256) ||
        ensure(x, x->totals, 256) || ensure(x, x->rng, 256) || ensure(x, x->bounds, 256) ||
        ensure(x, x->vtmp, 256))
        return fail(HHT_ENOMEM);
    if (cudaMallocHost((void**)&x->totals_h, sizeof(Totals)) != cudaSuccess ||
        cudaMallocHost((void**)&x->range_h, sizeof(RangeInfo)) != cudaSuccess ||
        cudaMallocHost((void**)&x->misc_h, 64) != cudaSuccess ||
        cudaMallocHost((void**)&x->pin, kPinBytes) != cudaSuccess ||
        cudaMallocHost((void**)&x->fin_h, kFinishBytes) != cudaSuccess)
        return fail(HHT_ECUDA);
    if (cudaHostGetDevicePointer((void**)&x->totals_m, x->totals_h, 0) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&x->range_m, x->range_h, 0) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&x->misc_m, x->misc_h, 0) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&x->fin_m, x->fin_h, 0) != cudaSuccess)
        return fail(HHT_ECUDA);
    x->group = o.group;
    if (o.nccl_comm) {   // the caller's communicator (borrowed)
        int cnt = 0, rk = 0;
        if (ncclCommCount((ncclComm_t)o.nccl_comm, &cnt) != ncclSuccess ||
            ncclCommUserRank((ncclComm_t)o.nccl_comm, &rk) != ncclSuccess)
            return fail(HHT_ENCCL);
        if (cnt != o.world || rk != o.rank) return fail(HHT_EINVAL);
        x->comm = (ncclComm_t)o.nccl_comm;
        x->own_comm = false;
    } else if (o.nccl_id) {   // world > 1, or world == 1 with an id: every collective runs (1-rank comm)
        ncclUniqueId id;
        memcpy(&id, o.nccl_id, sizeof id);
        if (ncclCommInitRank(&x->comm, o.world, id, o.rank) != ncclSuccess) return fail(HHT_ENCCL);
    }
    if (cudaStreamSynchronize(x->st) != cudaSuccess) return fail(HHT_ECUDA);
    *out = x;
    return HHT_OK;
}

hht_status hht_detect(hht_ctx* ctx, const int32_t* points, int64_t n, int32_t N, int32_t depth, int64_t threshold) {
    if (!ctx) return HHT_EINVAL;
    if (n < 0) return set_err(ctx, HHT_EINVAL, "n < 0");
    const int64_t off[2] = {0, n};
    return detect_impl(ctx, points, off, 1, N, depth, threshold);
}

hht_status hht_detect_batch(hht_ctx* ctx, const int32_t* points, const int64_t* offsets, int32_t B, int32_t N,
                            int32_t depth, int64_t threshold) {
    if (!ctx) return HHT_EINVAL;
    return detect_impl(ctx, points, offsets, B, N, depth, threshold);
}

hht_status hht_detect_trees(hht_ctx* ctx, const int32_t* points, const int64_t* tree_offsets, int32_t B, int32_t N,
                            int32_t depth, int64_t threshold) {
    if (!ctx) return HHT_EINVAL;
    if (!tree_offsets) return set_err(ctx, HHT_EINVAL, "tree_offsets is NULL");
    return detect_impl(ctx, points, nullptr, B, N, depth, threshold, tree_offsets);
}

hht_status hht_detect_image(hht_ctx* x, const uint8_t* img, int32_t N, int32_t mag_threshold, int32_t depth,
                            int64_t threshold) {
    if (!x) return HHT_EINVAL;
    x->err.clear();
    x->have = false;
    x->edges_valid = false;
    if (!img) return set_err(x, HHT_EINVAL, "img is NULL");
    if (N < 3 || N > 46340) return set_err(x, HHT_EINVAL, "image side must be in [3, 46340]");
    if (mag_threshold < 0) return set_err(x, HHT_EINVAL, "mag_threshold < 0");
    if (multi(x)) return set_err(x, HHT_EINVAL, "hht_detect_image runs on one rank (shard with hht_detect_trees)");
    CK(cudaSetDevice(x->opts.device));
    const uint64_t npix = (uint64_t)N * N;
    const uint8_t* dimg = img;
    cudaPointerAttributes pa{};
    cudaError_t e = cudaPointerGetAttributes(&pa, img);
    if (e != cudaSuccess) cudaGetLastError();
    if (!(e == cudaSuccess && (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged))) {
        TRY(ensure(x, x->img, npix));
        CK(cudaMemcpyAsync(x->img.p, img, npix, cudaMemcpyHostToDevice, x->st));
        dimg = (const uint8_t*)x->img.p;
    }
    const uint32_t ntiles = (uint32_t)((npix + kEdgeTile - 1) / kEdgeTile);
    TRY(ensure(x, x->packed, npix * 4));
    TRY(ensure(x, x->edgeB, npix * 4));
    // header (ticket at 0, super-tile sums at 2048) | tile words | (rows of 16k pixels: one mask word
    // per thread of the mask pass)
    constexpr size_t kEdgeHdr = 4096;
    TRY(ensure(x, x->edgetiles, kEdgeHdr + (size_t)ntiles * 8 + (size_t)ntiles * 256 * 4));
    CK(cudaMemsetAsync(x->edgetiles.p, 0, kEdgeHdr + (N % 16 != 0 ? (size_t)ntiles * 8 : 0), x->st));
    uint32_t super_shift = 7;
    while ((ntiles >> super_shift) >= 256) ++super_shift;
    EdgeArgs a{};
    a.img = dimg;
    a.W = a.H = N;
    a.thr = mag_threshold;
    a.outA = (uint32_t*)x->packed.p;
    a.outB = (uint32_t*)x->edgeB.p;
    a.tiles = (unsigned long long*)((char*)x->edgetiles.p + kEdgeHdr);
    a.supers = (unsigned long long*)((char*)x->edgetiles.p + 2048);
    a.super_shift = super_shift;
    a.tile_ctr = (uint32_t*)x->edgetiles.p;
    a.ntiles = ntiles;
    a.masks = (uint32_t*)((char*)x->edgetiles.p + kEdgeHdr + (size_t)ntiles * 8);
    a.totals = x->misc_m;
    CK(cudaEventRecord(x->ee0, x->st));
    CK(launch_edges(a, x->st));
    CK(cudaEventRecord(x->ee1, x->st));
    TRY(sync(x));
    float edge_ms = 0;
    CK(cudaEventElapsedTime(&edge_ms, x->ee0, x->ee1));
    const int64_t na = (int64_t)x->misc_h[0], nb = (int64_t)x->misc_h[1];
    // the trees' point sets, contiguous in x->packed: ALPHA points, then BETA points
    const bool wa = x->opts.halves & HHT_ALPHA, wb = x->opts.halves & HHT_BETA;
    int64_t toff[3] = {0, 0, 0};
    int k = 0;
    if (wa) toff[++k] = na;
    if (wb) {
        CK(cudaMemcpyAsync((uint32_t*)x->packed.p + (wa ? na : 0), x->edgeB.p, (size_t)nb * 4,
                           cudaMemcpyDeviceToDevice, x->st));
        toff[k + 1] = toff[k] + nb;
    }
    TRY(detect_impl(x, (const int32_t*)x->packed.p, nullptr, 1, N, depth, threshold, toff, true));
    x->edge_na = wa ? na : 0;
    x->edge_nb = wb ? nb : 0;
    x->edges_valid = true;
    if (x->opts.profile) {            // the detection reset the profile: add the edge kernel (class 0)
        x->prof.launches[0] += 1;
        x->prof.ms[0] += edge_ms;
        x->prof.bytes[0] += npix + 4ull * (uint64_t)(na + nb);
    }
    return HHT_OK;
}

hht_status hht_result_edges(hht_ctx* x, int32_t* out, int64_t cap, int64_t* n_alpha, int64_t* n_beta) {
    if (!x || !n_alpha || !n_beta) return HHT_EINVAL;
    if (!x->edges_valid) return set_err(x, HHT_ESTATE, "no hht_detect_image result");
    *n_alpha = x->edge_na;
    *n_beta = x->edge_nb;
    const int64_t n = x->edge_na + x->edge_nb;
    if (!out) return HHT_OK;
    if (cap < n) return set_err(x, HHT_EINVAL, "cap < %lld edge points", (long long)n);
    std::vector<uint32_t> h((size_t)n);
    if (n) CK(cudaMemcpyAsync(h.data(), x->packed.p, (size_t)n * 4, cudaMemcpyDeviceToHost, x->st));
    TRY(sync(x));
    for (int64_t i = 0; i < n; ++i) {
        out[2 * i] = (int32_t)(h[i] >> 16);
        out[2 * i + 1] = (int32_t)(h[i] & 0xFFFFu);
    }
    return HHT_OK;
}

// solution() with removal (NEXT-1) over the last detect's candidate leaves; cached until the next detect.
// One cooperative kernel per group of trees (k_rm, see hht_kernels.cu): live vote counts per candidate,
// a dense leaf-cell -> candidate map per tree of the group, removed flags per (tree, point).
hht_status compute_lines(hht_ctx* x) {
    if (x->lines_ok) return HHT_OK;
    if (multi(x)) return set_err(x, HHT_EINVAL, "removal needs every point of a tree: single rank only");
    if (x->circle) return set_err(x, HHT_EINVAL, "removal is defined for the exact test");
    TRY(host_leaves(x));
    const std::vector<LeafRec>& L = x->leaves_host;
    const uint32_t nt = (uint32_t)x->ntrees;
    std::vector<uint64_t> cand_lo(nt + 1, 0), rm_off(nt + 1, 0);
    {
        uint64_t k = 0;
        for (uint32_t t = 0; t < nt; ++t) {
            cand_lo[t] = k;
            while (k < L.size() && L[k].tree == t) ++k;
        }
        cand_lo[nt] = k;
        for (uint32_t t = 0; t < nt; ++t) rm_off[t + 1] = rm_off[t] + x->tree_pt_n[t];
    }
    const uint64_t ncand = L.size(), npts = rm_off[nt];
    const uint64_t per_tree = 4ull << (2 * x->D);                 // dense cell map of one tree
    const uint64_t fixed = ncand * 12 + npts * 25 + (uint64_t)nt * 48 + 4096;
    if (fixed + per_tree > x->budget)
        return set_err(x, HHT_ENOMEM, "removal post-pass needs %llu B (candidates, points and one 4^depth cell map)",
                       (unsigned long long)(fixed + per_tree));
    const uint32_t gmax = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(nt ? nt : 1, (x->budget - fixed) / per_tree));
    Buf big, meta;
    auto cleanup = [&]() { for (Buf* b : {&big, &meta}) if (b->p) cudaFreeAsync(b->p, x->st); };
    // big: live | out | out_live (ncand each) | queue (4 npts) | sup (2 npts) | removed (npts) | cellmap
    const uint64_t nc1 = std::max<uint64_t>(ncand, 1), np1 = std::max<uint64_t>(npts, 1);
    const uint64_t qwords = 4 * np1 + 2ull * (nt + 1) + 4;          // queue; later rows + line bases
    const uint64_t big_bytes = nc1 * 12 + qwords * 4 + np1 * 8 + ((np1 + 15) / 16) * 16 + (uint64_t)gmax * per_tree;
    hht_status st = ensure(x, big, big_bytes);
    if (st == HHT_OK) st = ensure(x, meta, (size_t)(nt + 1) * 8 * 3 + (size_t)nt * 16 + 64);
    if (st != HHT_OK) { cleanup(); return st; }
    uint32_t* d_live = (uint32_t*)big.p;
    uint32_t* d_out = d_live + nc1;
    uint32_t* d_out_live = d_out + nc1;
    uint32_t* d_queue = d_out_live + nc1;
    uint32_t* d_sup = d_queue + qwords;
    uint8_t* d_removed = (uint8_t*)(d_sup + 2 * np1);
    uint32_t* d_cellmap = (uint32_t*)(d_removed + ((np1 + 15) / 16) * 16);
    uint64_t* d_cand = (uint64_t*)meta.p;
    uint64_t* d_ptoff = d_cand + (nt + 1);
    uint64_t* d_rmoff = d_ptoff + (nt + 1);
    uint32_t* d_ptn = (uint32_t*)(d_rmoff + (nt + 1));
    uint32_t* d_cur = d_ptn + nt;
    uint32_t* d_pos = d_cur + nt;
    uint32_t* d_outn = d_pos + nt;
    uint32_t* d_small = d_outn + nt;                      // active[2], qn[2]
    unsigned long long* d_supn = (unsigned long long*)(d_small + 4);
    CK(cudaMemcpyAsync(d_cand, cand_lo.data(), (nt + 1) * 8, cudaMemcpyHostToDevice, x->st));
    if (nt) {
        CK(cudaMemcpyAsync(d_ptoff, x->tree_pt_off.data(), nt * 8, cudaMemcpyHostToDevice, x->st));
        CK(cudaMemcpyAsync(d_rmoff, rm_off.data(), nt * 8, cudaMemcpyHostToDevice, x->st));
        CK(cudaMemcpyAsync(d_ptn, x->tree_pt_n.data(), nt * 4, cudaMemcpyHostToDevice, x->st));
    }
    CK(cudaMemsetAsync(d_cur, 0, (size_t)nt * 12 + 16 + 8, x->st));       // cur, pos, out_n, small, sup_n
    CK(cudaMemsetAsync(d_removed, 0, np1, x->st));
    RmArgs a{};
    a.leaves = (const LeafRec*)x->leaves.b.p;
    a.cand_lo = d_cand;
    a.packed = (const uint32_t*)x->packed.p;
    a.pt_off = d_ptoff;
    a.pt_n = d_ptn;
    a.rm_off = d_rmoff;
    a.tree_beta = (const uint8_t*)x->beta.p;
    a.live = d_live;
    a.cellmap = d_cellmap;
    a.removed = d_removed;
    a.queue = d_queue;
    a.queue_cap = np1;
    a.qn = d_small + 2;
    a.cur = d_cur;
    a.pos = d_pos;
    a.active = d_small;
    a.out = d_out;
    a.out_live = d_out_live;
    a.out_n = d_outn;
    a.sup = d_sup;
    a.sup_n = d_supn;
    a.N = x->N;
    a.D = x->D;
    a.T = x->T;
    if (!x->rm_grid[x->int64 ? 1 : 0]) x->rm_grid[x->int64 ? 1 : 0] = x->sms * rm_blocks_per_sm(x->int64);
    for (uint32_t t0 = 0; t0 < nt; t0 += gmax) {
        a.t0 = t0;
        a.t1 = std::min(nt, t0 + gmax);
        if (cand_lo[a.t1] == cand_lo[t0]) continue;       // no candidates: nothing to emit
        CK(cudaMemsetAsync(d_cellmap, 0xFF, (size_t)(a.t1 - t0) * per_tree, x->st));
        CK(launch_removal(a, (const LeafRec*)x->leaves.b.p, x->int64, x->rm_grid[x->int64 ? 1 : 0], x->st));
    }
    std::vector<uint32_t> h_n(nt);
    unsigned long long h_supn = 0;
    if (nt) CK(cudaMemcpyAsync(h_n.data(), d_outn, nt * 4, cudaMemcpyDeviceToHost, x->st));
    CK(cudaMemcpyAsync(&h_supn, d_supn, 8, cudaMemcpyDeviceToHost, x->st));
    TRY(sync(x));
    std::vector<uint64_t> line_base(nt + 1, 0);
    for (uint32_t t = 0; t < nt; ++t) line_base[t + 1] = line_base[t] + h_n[t];
    const uint64_t nlines = line_base[nt];
    // rows (5 u32) and line bases reuse the queue area (qwords >= 5 nlines + 2 (nt + 1) + 2, since a
    // line removes more than T >= 1 points: nlines <= npts / 2)
    uint32_t* d_rows = d_queue;
    uint64_t* d_lbase = (uint64_t*)(((uintptr_t)(d_rows + 5 * nlines) + 7) & ~(uintptr_t)7);
    CK(cudaMemcpyAsync(d_lbase, line_base.data(), (nt + 1) * 8, cudaMemcpyHostToDevice, x->st));
    if (ncand) CK(launch_rm_rows((const LeafRec*)x->leaves.b.p, d_cand, d_out, d_out_live, d_outn, d_lbase,
                                 (const uint8_t*)x->beta.p, nt, (uint32_t)x->H, ncand, d_rows, d_sup, h_supn, x->st));
    x->lines_host.resize(nlines);
    std::vector<uint32_t> h_sup(2 * h_supn);
    if (nlines) CK(cudaMemcpyAsync(x->lines_host.data(), d_rows, nlines * sizeof(hht_leaf), cudaMemcpyDeviceToHost, x->st));
    if (h_supn) CK(cudaMemcpyAsync(h_sup.data(), d_sup, 8ull * h_supn, cudaMemcpyDeviceToHost, x->st));
    TRY(sync(x));
    cleanup();
    x->lines_img.assign(x->B + 1, 0);
    for (uint32_t t = 0; t < nt; ++t) x->lines_img[t / x->H + 1] = (int64_t)line_base[t + 1];
    for (int b = 1; b <= x->B; ++b) x->lines_img[b] = std::max(x->lines_img[b], x->lines_img[b - 1]);
    // supports as (line, point); sorted by line then point on first request (hht_result_line_points)
    x->lines_sup.resize(h_supn);
    for (uint64_t s = 0; s < h_supn; ++s) x->lines_sup[s] = {(uint64_t)h_sup[2 * s], h_sup[2 * s + 1]};
    x->lines_sup_sorted = false;
    x->lines_ok = true;
    return HHT_OK;
}

hht_status hht_result_lines(hht_ctx* x, int32_t image, hht_leaf* out, int64_t cap, int64_t* count) {
    if (!x || !count) return HHT_EINVAL;
    if (!x->have) return set_err(x, HHT_ESTATE, "no successful detect yet");
    if (image < -1 || image >= x->B) return set_err(x, HHT_EINVAL, "image out of range");
    TRY(compute_lines(x));
    const int64_t b = image < 0 ? 0 : x->lines_img[image], e = image < 0 ? (int64_t)x->lines_host.size()
                                                                        : x->lines_img[image + 1];
    *count = e - b;
    if (!out) return HHT_OK;
    if (cap < e - b) return set_err(x, HHT_EINVAL, "cap < %lld lines", (long long)(e - b));
    if (e > b) memcpy(out, x->lines_host.data() + b, (size_t)(e - b) * sizeof(hht_leaf));
    return HHT_OK;
}

hht_status hht_result_line_points(hht_ctx* x, int32_t image, uint32_t* out, int64_t cap, int64_t* count) {
    if (!x || !count) return HHT_EINVAL;
    if (!x->have) return set_err(x, HHT_ESTATE, "no successful detect yet");
    if (image < -1 || image >= x->B) return set_err(x, HHT_EINVAL, "image out of range");
    TRY(compute_lines(x));
    const uint64_t lb = image < 0 ? 0 : (uint64_t)x->lines_img[image];
    const uint64_t le = image < 0 ? x->lines_host.size() : (uint64_t)x->lines_img[image + 1];
    if (!x->lines_sup_sorted) {
        std::sort(x->lines_sup.begin(), x->lines_sup.end());
        x->lines_sup_sorted = true;
    }
    const auto& S = x->lines_sup;
    const auto lo = std::lower_bound(S.begin(), S.end(), std::make_pair(lb, 0u));
    const auto hi = std::lower_bound(S.begin(), S.end(), std::make_pair(le, 0u));
    *count = hi - lo;
    if (!out) return HHT_OK;
    if (cap < *count) return set_err(x, HHT_EINVAL, "cap < %lld support rows", (long long)*count);
    int64_t k = 0;
    for (auto it = lo; it != hi; ++it, ++k) {
        out[2 * k] = (uint32_t)(it->first - lb);
        out[2 * k + 1] = it->second;
    }
    return HHT_OK;
}

hht_status hht_result_leaves(hht_ctx* x, int32_t image, hht_leaf* out, int64_t cap, int64_t* count) {
    if (!x || !count) return HHT_EINVAL;
    if (!x->have) return set_err(x, HHT_ESTATE, "no successful detect yet");
    if (image < -1 || image >= x->B) return set_err(x, HHT_EINVAL, "image out of range");
    if (image == -1) {
        // every leaf: convert on the device, then one copy into the caller's buffer
        *count = (int64_t)x->leaves.n;
        if (cap < *count) return set_err(x, HHT_EINVAL, "cap %lld < %lld leaves", (long long)cap, (long long)*count);
        if (!*count) return HHT_OK;
        if (!out) return set_err(x, HHT_EINVAL, "out is NULL");
        TRY(ensure(x, x->leafrows, x->leaves.n * sizeof(hht_leaf)));
        CK(launch_leaf_rows((const LeafRec*)x->leaves.b.p, x->leaves.n, (const uint8_t*)x->beta.p, x->H,
                            (uint32_t*)x->leafrows.p, x->st));
        CK(cudaMemcpyAsync(out, x->leafrows.p, x->leaves.n * sizeof(hht_leaf), cudaMemcpyDefault, x->st));
        TRY(sync(x));
        x->stat.d2h_bytes += x->leaves.n * sizeof(hht_leaf);
        return HHT_OK;
    }
    TRY(host_leaves(x));
    const auto& L = x->leaves_host;
    uint64_t b = 0, e = L.size();
    if (image >= 0) {
        const uint32_t t0 = (uint32_t)image * x->H, t1 = t0 + x->H;
        b = std::lower_bound(L.begin(), L.end(), t0, [](const LeafRec& r, uint32_t t) { return r.tree < t; }) - L.begin();
        e = std::lower_bound(L.begin(), L.end(), t1, [](const LeafRec& r, uint32_t t) { return r.tree < t; }) - L.begin();
    }
    *count = (int64_t)(e - b);
    if (cap < *count) return set_err(x, HHT_EINVAL, "cap %lld < %lld leaves", (long long)cap, (long long)*count);
    if (!*count) return HHT_OK;
    if (!out) return set_err(x, HHT_EINVAL, "out is NULL");
    std::vector<hht_leaf> tmp(e - b);
    for (uint64_t k = b; k < e; ++k) {
        const LeafRec& r = L[k];
        tmp[k - b] = {(int32_t)(r.tree / x->H), x->tree_half[r.tree], r.i, r.j, r.votes};
    }
    CK(cudaMemcpy(out, tmp.data(), tmp.size() * sizeof(hht_leaf), cudaMemcpyDefault));
    return HHT_OK;
}

hht_status hht_result_level(hht_ctx* x, int32_t image, uint32_t half, int32_t level, uint32_t* out, int64_t cap,
                            int64_t* count) {
    if (!x || !count) return HHT_EINVAL;
    if (!x->have) return set_err(x, HHT_ESTATE, "no successful detect yet");
    if (!x->opts.record_levels) return set_err(x, HHT_ESTATE, "record_levels is off");
    if (image < 0 || image >= x->B) return set_err(x, HHT_EINVAL, "image out of range");
    if (level < 0 || level > x->D) return set_err(x, HHT_EINVAL, "level out of range");
    if (!(half == HHT_ALPHA || half == HHT_BETA) || !(x->opts.halves & half)) return set_err(x, HHT_EINVAL, "half not computed");
    const uint32_t t = (uint32_t)image * x->H + ((half == HHT_BETA && (x->opts.halves & HHT_ALPHA)) ? 1 : 0);
    TRY(host_records(x, level));
    const auto& R = x->rec_host[level];
    const auto lo = std::lower_bound(R.begin(), R.end(), t, [](const Record& r, uint32_t v) { return r.tree < v; });
    const auto hi = std::lower_bound(R.begin(), R.end(), t + 1, [](const Record& r, uint32_t v) { return r.tree < v; });
    *count = (int64_t)(hi - lo);
    if (cap < *count) return set_err(x, HHT_EINVAL, "cap %lld < %lld records", (long long)cap, (long long)*count);
    if (!*count) return HHT_OK;
    if (!out) return set_err(x, HHT_EINVAL, "out is NULL");
    std::vector<uint32_t> tmp(3 * (size_t)*count);
    size_t k = 0;
    for (auto it = lo; it != hi; ++it) {
        tmp[k++] = it->a;
        tmp[k++] = it->c;
        tmp[k++] = it->votes;
    }
    CK(cudaMemcpy(out, tmp.data(), tmp.size() * 4, cudaMemcpyDefault));
    return HHT_OK;
}

static hht_status set_sink(hht_ctx* x, void* host, int64_t cap, bool packed) {
    if (!x) return HHT_EINVAL;
    if (host && cap < 0) return set_err(x, HHT_EINVAL, "cap < 0");
    if (x->cst) cudaStreamSynchronize(x->cst);
    for (int k = 0; k < kSinkSlots; ++k) x->copy_pending[k] = false;
    x->sink = host;
    x->sink_packed = host && packed;
    x->sink_cap = host ? cap : 0;
    return HHT_OK;
}

hht_status hht_set_leaf_sink(hht_ctx* x, hht_leaf* host, int64_t cap) { return set_sink(x, host, cap, false); }

hht_status hht_set_leaf_sink_packed(hht_ctx* x, uint64_t* host, int64_t cap) { return set_sink(x, host, cap, true); }

hht_status hht_result_tree_offsets(hht_ctx* x, uint64_t* out, int64_t cap, int64_t* ntrees) {
    if (!x || !ntrees) return HHT_EINVAL;
    if (!x->have) return set_err(x, HHT_ESTATE, "no successful detect yet");
    *ntrees = x->ntrees;
    if (!out) return HHT_OK;
    if (cap < (int64_t)x->ntrees + 1) return set_err(x, HHT_EINVAL, "cap %lld < %d tree offsets", (long long)cap, x->ntrees + 1);
    TRY(ensure(x, x->treeoff, 8ull * (x->ntrees + 1)));
    CK(launch_tree_offsets((const LeafRec*)x->leaves.b.p, x->leaves.n, (uint32_t)x->ntrees, (uint64_t*)x->treeoff.p, x->st));
    CK(cudaMemcpyAsync(out, x->treeoff.p, 8ull * (x->ntrees + 1), cudaMemcpyDefault, x->st));
    return sync(x);
}

hht_status hht_result_stats(hht_ctx* x, hht_stats* out) {
    if (!x || !out) return HHT_EINVAL;
    if (!x->have) return set_err(x, HHT_ESTATE, "no successful detect yet");
    *out = x->stat;
    return HHT_OK;
}

hht_status hht_result_profile(hht_ctx* x, hht_profile* out) {
    if (!x || !out) return HHT_EINVAL;
    if (!x->have) return set_err(x, HHT_ESTATE, "no successful detect yet");
    *out = x->prof;
    return HHT_OK;
}

hht_status hht_result_launches(hht_ctx* x, hht_launch* out, int64_t cap, int64_t* count) {
    if (!x || !count) return HHT_EINVAL;
    if (!x->have) return set_err(x, HHT_ESTATE, "no successful detect yet");
    *count = (int64_t)x->launch_log.size();
    if (cap < *count) return set_err(x, HHT_EINVAL, "cap %lld < %lld launches", (long long)cap, (long long)*count);
    if (*count && !out) return set_err(x, HHT_EINVAL, "out is NULL");
    for (int64_t i = 0; i < *count; ++i) out[i] = x->launch_log[i];
    return HHT_OK;
}

hht_status hht_timer_begin(hht_ctx* x) {
    if (!x) return HHT_EINVAL;
    CK(cudaEventRecord(x->tb0, x->st));
    return HHT_OK;
}

hht_status hht_timer_end(hht_ctx* x, double* ms) {
    if (!x || !ms) return HHT_EINVAL;
    CK(cudaEventRecord(x->tb1, x->st));
    CK(cudaEventSynchronize(x->tb1));
    float m = 0;
    CK(cudaEventElapsedTime(&m, x->tb0, x->tb1));
    *ms = m;
    return HHT_OK;
}

const char* hht_last_error(const hht_ctx* x) { return x ? x->err.c_str() : "null context"; }

void hht_destroy(hht_ctx* x) {
    if (!x) return;
    if (x->st) cudaStreamSynchronize(x->st);
    if (x->cst) cudaStreamSynchronize(x->cst);
    for (Buf& b : x->sinkrows)
        if (b.p) cudaFree(b.p);
    for (int k = 0; k < kSinkSlots; ++k) {
        if (x->ev_conv[k]) cudaEventDestroy(x->ev_conv[k]);
        if (x->ev_copy[k]) cudaEventDestroy(x->ev_copy[k]);
    }
    if (x->cst) cudaStreamDestroy(x->cst);
    if (x->cst2) { cudaStreamSynchronize(x->cst2); cudaStreamDestroy(x->cst2); }
    if (x->ev_tail) cudaEventDestroy(x->ev_tail);
    if (x->ev_ar) cudaEventDestroy(x->ev_ar);
    for (Buf* b : {&x->dense2[0], &x->dense2[1]})
        if (b->p) cudaFree(b->p);
    auto fr = [&](Buf& b) {
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
    };
    for (auto& L : x->lv) {
        for (Buf* b : {&L.tree, &L.a, &L.c, &L.parent, &L.len, &L.votes_g, &L.off, &L.choff, &L.chunks, &L.nf, &L.nfoff, &L.votes,
                       &L.votes_local, &L.cursor, &L.list_own})
            fr(*b);
    }
    for (auto& g : x->rec) fr(g.b);
    fr(x->leaves.b);
    for (Buf* b : {&x->stage_in, &x->packed, &x->errflag, &x->beta, &x->stats, &x->tiles, &x->tilectr, &x->totals,
                   &x->rng, &x->bounds, &x->vtmp, &x->dense, &x->gv, &x->leafrows, &x->treeoff, &x->fusedctr, &x->img, &x->units,
                   &x->edgeB, &x->edgetiles, &x->small, &x->small_g})
        fr(*b);
    if (x->totals_h) cudaFreeHost(x->totals_h);
    if (x->range_h) cudaFreeHost(x->range_h);
    if (x->misc_h) cudaFreeHost(x->misc_h);
    if (x->pin) cudaFreeHost(x->pin);
    if (x->fin_h) cudaFreeHost(x->fin_h);
    for (auto& e : x->pev) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    for (cudaEvent_t e : {x->ev0, x->ev1, x->tb0, x->tb1, x->ee0, x->ee1})
        if (e) cudaEventDestroy(e);
    if (x->comm && x->own_comm) ncclCommDestroy(x->comm);
    if (x->own_st) cudaStreamDestroy(x->own_st);
    delete x;
}

hht_status hht_set_stream(hht_ctx* x, void* stream) {
    if (!x) return HHT_EINVAL;
    const cudaStream_t next = stream ? (cudaStream_t)stream : x->own_st;
    if (next == x->st) return HHT_OK;
    CK(cudaStreamSynchronize(x->st));
    x->st = next;
    return HHT_OK;
}

}  // extern "C"

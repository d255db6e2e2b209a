// Internal interface between the level driver (hht_driver.cu) and the kernels (hht_kernels.cu).
// Not part of the C ABI. Nothing here is shared with oracle/.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hht {

constexpr int kWarp = 32;
constexpr int kItems = 8;                  // list entries per lane per chunk
constexpr int kChunk = kWarp * kItems;     // 256 entries: one warp work unit, never spans regions
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kSplitThreads = 256;         // split kernel: one thread per parent (its 4 children)
constexpr int kTailCells = 64;             // 8x8 tail: leaf grid per level-(D-3) region
constexpr int kTail16Cells = 256;          // 16x16 tail: leaf grid per level-(D-4) region

// Quad order of the paper: q = 0 NE, 1 NW, 2 SW, 3 SE; child (2a+da, 2c+dc).
__host__ __device__ constexpr uint32_t quad_da(int q) { return (q == 0 || q == 3) ? 1u : 0u; }
__host__ __device__ constexpr uint32_t quad_dc(int q) { return (q <= 1) ? 1u : 0u; }

// One warp work unit of a pass: <= kChunk consecutive entries of ONE region's candidate list, with
// everything the pass needs about the region, so that a chunk costs one 32-byte load before its
// entries can be fetched (and that load is issued one chunk ahead).
struct alignas(16) ChunkDesc {
    uint32_t r;          // region index in its level's frontier
    uint32_t cnt;        // entries in this chunk (1..kChunk)
    uint32_t a, c;       // region lattice coordinates
    uint64_t e0;         // absolute list offset of the first entry
    uint32_t beta;       // 1 = BETA tree (swap x and y)
    uint32_t pad;
};

// Frontier of split regions at one level, structure of arrays in HBM.
struct Frontier {
    uint32_t* tree;      // tree id (image * H + half index)
    uint32_t* a;         // region column (m axis)
    uint32_t* c;         // region row (b axis)
    uint32_t* parent;    // index of the parent in the previous level's frontier
    uint32_t* len;       // local votes = local candidate-list length (this rank's lines crossing it)
    uint32_t* votes;     // global votes (all ranks)
    uint64_t* off;       // [F+1] local list offset (exclusive scan of len); off[F] = total
    uint64_t* choff;     // [F+1] chunk offset (exclusive scan of ceil(len/kChunk)); choff[F] = total
    ChunkDesc* chunks;   // [total chunks] work-unit descriptors (k_chunk_map)
};

struct alignas(16) Record { uint32_t tree, a, c, votes; };     // one visited region
struct alignas(16) LeafRec { uint32_t tree, i, j, votes; };     // one detected line

// Look-back tile descriptor for the split scan (status: 0 none, 1 aggregate, 2 inclusive prefix).
struct TileDesc {
    uint32_t status;
    uint32_t aggF, aggC, pad0;
    uint64_t aggS;
    uint32_t incF, incC;
    uint64_t incS;
};

struct Totals {          // written by the last split tile
    uint64_t F, S, C;
};

// Device-side stats accumulators (uint64): see kStat*.
enum { kStatTests = 0, kStatVotes = 1, kStatLeaves = 2, kStatSplit0 = 8, kStatVisited0 = 8 + 64,
       kStatCount = 8 + 128 };
// The one-launch paths' mapped host block (SmallArgs / MidArgs::fin), written by the kernel itself:
// word 0 the range flag, words 1.. the per-level counts (<= 64 + 2), from word kFinishStatsWord the
// statistics (kStatCount u64)
constexpr uint32_t kFinishStatsWord = 128;
constexpr size_t kFinishBytes = kFinishStatsWord * 4 + kStatCount * 8;

enum PassMode { MODE_COUNT = 0, MODE_WRITE = 1, MODE_COUNT2 = 2, MODE_WRITE_NC = 3 };   // NC: no count-ahead

// Geometry of one pass over the lists of split regions at parent level l:
//   g(p) = G(i0, j0) = ex*alpha + (ey << D) + beta,  alpha = 2^D - 2*i0,  beta = N*2^D - 3N*j0,
//   child SW values g - {0,Pc} - {0,Qc}, Pc = ex << (D-l), Qc = 3N*2^(D-l-1); child votes iff
//   0 < g_child <= Pc + Qc; grandchildren likewise with Pg = Pc/2, Qg = Qc/2.
struct PassArgs {
    // parent level
    const uint32_t* list;          // packed (x << 16 | y) candidate lines of the parents
    uint64_t list_base;            // subtract from ChunkDesc::e0 to index `list`
    const ChunkDesc* chunks;       // parents' chunk descriptors
    const uint64_t* chunk_bounds;  // device [2]: chunk range [lo, hi) of this launch
    int level;                     // parent level l
    int D;
    int N;
    // children of the parents (level l+1)
    const uint32_t* nf;            // [4 * nparents] child -> next-frontier index or kNone
    const uint64_t* nfoff;         // [4 * nparents] list offset of each split child (next frontier)
    uint32_t nf_rbase;             // parent index of nf[0..3]
    uint32_t q0, q1;               // only next-frontier indices in [q0, q1) are written / counted
    uint64_t c_list_base;          // subtract from nfoff[] to index c_list
    uint32_t* c_cursor;            // [q1 - q0] append cursors
    uint32_t* c_list;              // output lists
    uint32_t one;                  // == 1 (runtime value: keeps the count adds on the FMA pipe)
    uint32_t fx_m, fx_mlo, fx_s;   // 16x16 raster fixed point: ceil / floor(2^(24+fx_s) / 3N), 2^fx_s >= 96N
    uint32_t* votes;               // MODE_COUNT: [4 * nparents] (4*(r - nf_rbase) + q)
                                   // else:       [4 * (q1 - q0)] (4*(nf - q0) + q')
                                   // tails: 256-cell leaf grids per region
    // fused tail (k_fused): parents R_l[r_lo, r_hi) are the work units, taken by warps from `work`
    const uint64_t* p_choff;       // parents' chunk offsets (their chunks are consecutive)
    uint32_t r_lo, r_hi;
    uint32_t* work;                // device counter, zero at launch
    unsigned long long* child_pairs;   // device counters: [0] (line, child) pairs rastered, [1] entries streamed
    uint32_t all_children;         // k_fused: raster all 4 children of every parent, grid 4 (r - r_lo) + q
    // k_fused from the grandparents' lists (tail_depth 6): work unit r of level l streams the list of
    // its parent gp_parent[r] (level l-1 chunks/lists above) and takes its region from gp_a/gp_c;
    // entries that do not cross r have no child bit set. nullptr: r's own list.
    const uint32_t* gp_parent;
    const uint32_t* gp_a;
    const uint32_t* gp_c;
    // k_fused with split work units (fewer parents than warps x kUnitsPerWarp): unit u = (r, k) covers
    // chunks [c_lo + k K, min(c_hi, c_lo + (k + 1) K)) of parent r, K = *unit_k (k_units); nullptr:
    // one unit per parent
    const uint2* units;
    const uint32_t* nunits;
    const uint32_t* unit_k;
};
constexpr uint32_t kUnitWhole = 0xFFFFFFFFu;   // work unit = the whole parent (k_units with k_split)
cudaError_t launch_units(const uint64_t* p_choff, uint32_t r_lo, uint32_t r_hi, uint32_t target_units, uint32_t r_split,
                         uint32_t k_split, uint2* units, uint32_t* nunits_k, cudaStream_t st);

struct SplitArgs {
    const uint32_t* V;             // [4 * Fp] global child votes
    const uint32_t* VL;            // [4 * Fp] local child votes (list lengths on this rank)
    uint32_t Fp;
    const uint32_t* p_tree;        // parent arrays, already offset to the range start
    const uint32_t* p_a;
    const uint32_t* p_c;
    uint32_t parent_base;          // global index of p_*[0]
    int child_level;
    int leaf_level;                // child_level == D: emit leaves, no frontier
    int need_lists;                // child_level <= D-2: children will carry candidate lists
    int write_off;                 // write the children's list lengths, votes and list / chunk
                                   // offsets (read by list passes, chunk maps, range selection and
                                   // the derived-NE split: list levels and D-1); other levels skip
                                   // 24 B per child
    int record;
    uint64_t T;
    const uint32_t* p_votes;       // derive_ne: parents' global votes (range start)
    const uint32_t* p_len;         // derive_ne: parents' local votes (range start)
    int derive_ne;                 // V/VL hold no NE counts: NE = parent - SW (votes identity)
    uint32_t* nf;                  // [4 * Fp]
    uint64_t* nfoff;               // [4 * Fp] list offset of each split child (need_lists)
    Frontier out;
    Record* rec;                   // records of child_level, rec[4*p + q]
    LeafRec* leaves;               // leaves[leaf index]
    TileDesc* tiles;
    TileDesc* scan_seg;            // [kScanBlocks] segment descriptors of k_split_scan's look-back
    uint32_t* tile_counter;
    unsigned long long* stats;
    Totals* totals;
    uint32_t ntiles;
    int pass;                      // 0: single pass with look-back; 1: tile aggregates only;
                                   // 2: outputs, tiles[t].inc* = exclusive tile prefix (k_split_scan)
};

// Range selection over a next frontier (one thread).
struct RangeInfo {
    uint64_t q1;                   // proposed / final end of range
    uint64_t s_lo, s_hi;           // list offsets off[q0], off[q1]
    uint64_t chunk_lo, chunk_hi;   // parents' chunk bounds (written into chunk_bounds too)
    uint64_t pairs;                // parent entries streamed by this range's pass
};

// Launchers (hht_kernels.cu). All asynchronous on `st`.
cudaError_t launch_stage(const int32_t* pts, uint64_t n, int N, uint32_t* packed, uint32_t* err,
                         cudaStream_t st);
cudaError_t launch_pass(int mode, bool int64, int pf, int circle, const PassArgs& a, int grid, cudaStream_t st);
cudaError_t launch_split(const SplitArgs& a, int resident_blocks, cudaStream_t st);
int split_blocks_per_sm();
constexpr uint32_t kSplitPrescanTiles = 1024;   // reduce-then-scan split from this many tiles on
constexpr uint32_t kScanBlocks = 128;           // k_split_scan: at most this many segments (<= one block per SM)
cudaError_t launch_chunk_map(const uint64_t* choff, const uint64_t* off, const uint32_t* len, const uint32_t* a,
                             const uint32_t* c, const uint32_t* tree, const uint8_t* tree_beta, uint32_t F,
                             ChunkDesc* chunks, cudaStream_t st);
cudaError_t launch_range(const uint64_t* c_off, const uint32_t* c_parent, uint32_t Fc, uint32_t q0,
                         uint64_t cap_entries, uint64_t forced_q1, const uint64_t* p_off,
                         const uint64_t* p_choff, const uint32_t* p_len, int p_is_root, RangeInfo* info,
                         uint64_t* chunk_bounds, RangeInfo* info_h, cudaStream_t st);
cudaError_t launch_copy_u32(uint32_t* dst, const uint32_t* src, uint32_t n, cudaStream_t st);
cudaError_t launch_set_bounds(uint64_t* bounds, uint64_t lo, uint64_t hi, cudaStream_t st);
int pass_blocks_per_sm(int mode, bool int64, int pf, int circle);
int tail_blocks_per_sm(bool int64);
cudaError_t launch_leaf_packed(const LeafRec* in, uint64_t n, uint64_t* out, cudaStream_t st);
cudaError_t launch_tree_offsets(const LeafRec* in, uint64_t n, uint32_t ntrees, uint64_t* out, cudaStream_t st);
cudaError_t launch_leaf_rows(const LeafRec* in, uint64_t n, const uint8_t* tree_beta, uint32_t H, uint32_t* out,
                             cudaStream_t st);
cudaError_t launch_tail(bool int64, const PassArgs& a, int grid, cudaStream_t st);
struct GatherChain { const uint32_t* parent[3]; };   // parent-index arrays, nearest level first
cudaError_t launch_gather(const uint32_t* dense, uint32_t anc_base, const uint32_t* anc_a, const uint32_t* anc_c,
                          const uint32_t* p_a, const uint32_t* p_c, const GatherChain& chain, int hops, int tk,
                          int j, uint32_t Fp, uint32_t* V, const uint32_t* owner_parent, cudaStream_t st);
cudaError_t launch_grid_diag(const uint32_t* dense, uint32_t nparents, uint32_t* V, cudaStream_t st);
int tail16_blocks_per_sm(bool int64, bool pref);
cudaError_t launch_tail16(bool int64, bool pref, const PassArgs& a, int grid, cudaStream_t st);
int fused_blocks_per_sm(bool int64);
// Edge front end (k_edges): Sobel + L1 threshold + ALPHA/BETA partition, raster-order compaction.
struct EdgeArgs {
    const uint8_t* img;            // [H][W], row 0 = top
    int W, H, thr;
    uint32_t* outA;                // packed (x << 16 | y) ALPHA points, raster order
    uint32_t* outB;                // BETA points
    unsigned long long* tiles;     // [ntiles] k_edges: look-back words (zeroed); W % 16 == 0: tile counts (ALPHA << 32 | BETA)
    unsigned long long* supers;    // [<= 256] W % 16 == 0: sums of the tile counts per 2^super_shift tiles (zeroed)
    uint32_t super_shift;
    uint32_t* tile_ctr;            // zeroed (k_edges)
    uint32_t ntiles;               // 4096-pixel block tiles (k_edges)
    uint32_t* masks;               // [256 ntiles] W % 16 == 0: each thread's 16 edge bits | 16 ALPHA bits << 16
    uint64_t* totals;              // [2] (mapped host): ALPHA count, BETA count (written by the last tile)
};
constexpr int kEdgeTile = 4096;    // pixels per 256-thread tile (16 per lane, lane-interleaved)
cudaError_t launch_edges(const EdgeArgs& a, cudaStream_t st);
// solution() with point removal as a post-pass: per tree t, candidate leaves
// leaves[cand_lo[t] .. cand_lo[t+1]) and points packed[pt_off[t] .. pt_off[t] + pt_n[t]).
// solution() with removal (NEXT-1): cooperative greedy over the candidate leaves of trees [t0, t1)
constexpr int kRmThreads = 1024;
constexpr int kRmRedTrees = 16;          // k_rm: groups of at most this many trees search redundantly per block
constexpr int kRmCols = 8;               // k_rm: leaf columns rastered per thread and removed point
constexpr uint32_t kDone = 0xFFFFFFFEu;   // cur[t]: the tree's greedy has finished
struct RmArgs {
    const LeafRec* leaves;         // candidates (removal-off leaves), tree-major, depth-first order
    const uint64_t* cand_lo;       // [ntrees + 1]
    const uint32_t* packed;        // staged points
    const uint64_t* pt_off;        // [ntrees] tree t's points in packed
    const uint32_t* pt_n;          // [ntrees]
    const uint64_t* rm_off;        // [ntrees] tree t's removed flags in `removed`
    const uint8_t* tree_beta;
    uint32_t* live;                // [candidates] live votes
    uint32_t* cellmap;             // [(t1 - t0) 4^D] leaf cell -> candidate index within its tree, kNone
    uint8_t* removed;              // per (tree, point)
    uint32_t* queue;               // [2 rounds][queue_cap][2] (tree, point) removed in a round (parity)
    uint32_t* qn;                  // [2] queue counts by round parity
    uint64_t queue_cap;
    uint32_t* cur;                 // [ntrees] candidate emitted in the current round, kDone when finished
    uint32_t* pos;                 // [ntrees] next candidate to consider
    uint32_t* active;              // [2] trees that emitted in the round (round parity)
    uint32_t* out;                 // [candidates] emitted candidate indices, tree t's at cand_lo[t]
    uint32_t* out_live;            // live votes at emission
    uint32_t* out_n;               // [ntrees]
    uint32_t* sup;                 // [2 x points] (global line slot cand_lo[t] + e, point index in tree)
    unsigned long long* sup_n;
    int N, D;
    uint64_t T;
    uint32_t t0, t1;
};
int rm_blocks_per_sm(bool int64);
cudaError_t launch_rm_rows(const LeafRec* leaves, const uint64_t* cand_lo, const uint32_t* out, const uint32_t* out_live,
                           const uint32_t* out_n, const uint64_t* line_base, const uint8_t* tree_beta, uint32_t nt,
                           uint32_t H, uint64_t ncand, uint32_t* rows, uint32_t* sup, uint64_t nsup, cudaStream_t st);
cudaError_t launch_removal(const RmArgs& a, const LeafRec* leaves, bool int64, int grid, cudaStream_t st);
// Latency path (k_small): the whole level-synchronous traversal of a tiny detection in ONE block.
struct SmallArgs {
    uint32_t* packed;              // staged points (written here when `pts` is set)
    const int2* pts;               // non-null: raw device points [npts], staged and range-checked in the
    uint64_t npts;                 //   kernel (no separate stage launch); null: `packed` is already staged
    uint32_t* fin;                 // mapped host block (kFinish* layout): range flag, counts, statistics
    const uint64_t* tree_off;      // [ntrees] first point of each tree in `packed`
    const uint32_t* tree_n;        // [ntrees] points of each tree
    const uint8_t* tree_beta;
    uint32_t ntrees;
    int N, D;
    uint64_t T;
    // scratch (capacities from the host's bounds)
    uint32_t* list[2];             // global_scratch: the two candidate lists (list[1] = list[0] + smem_S);
                                   // the frontier arrays, votes and frontier indices are in shared memory
    // outputs
    Record* const* rec;            // [D + 1] per-level record arrays
    LeafRec* leaves;
    unsigned long long* stats;     // kStat* layout (tests, votes, leaves, split[l], visited[l])
    uint32_t* counts;              // [D + 2] records per level, then leaves (read by the host)
    uint32_t smem_S, smem_F;       // scratch capacities: list entries, frontier regions
    uint32_t global_scratch;       // 1: list[] are device (L2-resident) buffers set by the host, the
                                   //    frontier arrays stay in shared memory; 0: all in shared memory
};
uint64_t small_smem_bytes(uint32_t S, uint32_t F);
uint64_t small_frontier_bytes(uint32_t F);
constexpr uint64_t kSmallSmemMax = 220 * 1024;
#ifndef HHT_SMALL_GLOBAL_MAX_LOG2
#define HHT_SMALL_GLOBAL_MAX_LOG2 16
#endif
constexpr uint64_t kSmallGlobalMaxS = 1ull << HHT_SMALL_GLOBAL_MAX_LOG2;   // device-list latency path: list bound (entries)
cudaError_t launch_small(const SmallArgs& a, bool int64, cudaStream_t st);
// Mid-size latency path (hht_mid.cu): the whole traversal as one cooperative kernel over the GPU.
constexpr int kMidThreads = 256;
constexpr int kMidMinBlocks = 3;
constexpr uint32_t kMidMaxTiles = 3072;        // tiles of kMidThreads children per level (S2 prefixes)
constexpr uint64_t kMidMaxS = 1ull << 26;      // list bound (entries per level) admitted
struct MidArgs {
    uint32_t* packed;              // staged points (level-0 lists; written here when `pts` is set)
    const int2* pts;               // non-null: raw device points [npts], staged and range-checked in the
    uint64_t npts;                 //   kernel (no separate stage launch); null: `packed` is already staged
    uint32_t* fin;                 // mapped host block (kFinish* layout): range flag, counts, statistics
    const uint64_t* tree_off;      // [ntrees] first point of each tree in `packed`
    const uint32_t* tree_n;        // [ntrees]
    const uint8_t* tree_beta;
    uint32_t ntrees;
    int N, D;
    uint64_t T;
    uint32_t record;
    // scratch, double-buffered by level parity (capacities from the host's bounds)
    uint32_t* list[2];             // candidate lists (list[0] unused at level 0: the roots read `packed`)
    uint4* fd[2];                  // [2 F] region descriptors (tree | beta << 31, a, c, start), (len, coff)
    uint32_t* chunkmap[2];         // [chunks] chunk -> region (no search per work unit)
    uint32_t* cv[2];               // [4 F] votes of the frontier's children
    uint32_t* cursor;              // [4 F] child -> next-frontier index (tile-local flag scan in S1)
    uint32_t* loff;                // [4 F] tile-local list offsets
    uint32_t* lcoff;               // [4 F] tile-local chunk offsets
    uint32_t* app;                 // [F] append cursors of the next lists
    uint32_t* tiles;               // [3 x tiles] tile totals (split count, entries, chunks)
    uint32_t* ctl;                 // [8] per buffer: F, chunks, entries; ctl[3]: range flag (0 between calls)
    // outputs (as SmallArgs)
    Record* const* rec;
    LeafRec* leaves;
    unsigned long long* stats;
    uint32_t* counts;              // [D + 2] records per level, then leaves
};
int mid_blocks_per_sm(bool int64);
cudaError_t launch_mid(const MidArgs& a, bool int64, int grid, cudaStream_t st);
cudaError_t launch_fused(bool int64, const PassArgs& a, int grid, cudaStream_t st);
cudaError_t launch_bounds(const uint64_t* off, const uint64_t* choff, const uint32_t* len, uint32_t r0, uint32_t r1,
                          int is_root, RangeInfo* info, uint64_t* chunk_bounds, RangeInfo* info_h, cudaStream_t st);

}  // namespace hht

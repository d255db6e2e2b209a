/*
 * hht.h -- C ABI of libhht.so, a B200-native (sm_100a) implementation of the level-synchronous
 * hot path of Singh & Bhatia's hierarchical slope-intercept Hough transform with the exact 4-bit
 * corner-code membership test (arXiv 1007.0547; PAPER.md = the paper's text).
 *
 * What one detect call computes (§3 pseudocode, with getcode()
 * PAPER.md:146-164; readings R1-R16 in DESIGN.md §2):
 *   for every tree (image x half; ALPHA uses (x,y), BETA uses (y,x)) the quadtree over
 *   parameter space m in [-1,1] x b in [-N,2N] down to level `depth`; a region's votes are the
 *   number of edge points whose line b = y - x*m has a corner code other than 0000 and 1111 with
 *   respect to it; a region with votes > threshold is split into its four
 *   children NE, NW, SW, SE, which test only the lines that crossed it
 *   (PAPER.md:100-103); a level-`depth` region with votes > threshold is a detected line
 *   (solution() without point removal).
 *
 * Conventions shared by every call:
 *   - Every call returns hht_status; none throws, exits or prints. On error, hht_last_error(ctx)
 *     holds one line of text (CUDA / NCCL error strings included).
 *   - A ctx is not thread-safe: use one ctx per (host thread, device).
 *   - Point arrays are int32 (x, y) pairs, row-major [n][2], 8-byte aligned. They may be device
 *     memory (the fast path) or host memory (pageable or pinned: the library stages them with one
 *     host-to-device copy per call, counted in the result's h2d_bytes). They are borrowed for the
 *     duration of the call only; every detect call is synchronous on return.
 *   - Lattice: corners m_i = -1 + 2i/2^D, b_j = -N + 3N*j/2^D, i,j in [0, 2^D]; a level-l region
 *     (a, c) spans lattice [a*s, (a+1)*s] x [c*s, (c+1)*s] with s = 2^(D-l). A leaf (i, j) at level D
 *     covers m in [m_i, m_(i+1)], b in [b_j, b_(j+1)] -- exact dyadic rationals.
 *   - Outputs are owned by the ctx until the next detect call or hht_destroy; getters copy out
 *     to host OR device memory (cudaMemcpyDefault). A too-small `cap` returns HHT_EINVAL with
 *     *count set to the required number of elements.
 */
#ifndef HHT_H
#define HHT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HHT_OK = 0,
    HHT_EINVAL = 1,     /* null pointer, n < 0, N < 1 or N > 65536, depth < 1 or > 30, threshold < 1,
                           bad halves, unaligned points, bad image/half/level in a getter, small cap */
    HHT_ERANGE = 2,     /* a point outside [0,N)^2, found before any traversal */
    HHT_EOVERFLOW = 3,  /* 5*N*2^depth >= 2^62: exact int64 corner arithmetic impossible */
    HHT_ENOMEM = 4,     /* device memory budget cannot hold one region's candidate list */
    HHT_ECUDA = 5,      /* CUDA runtime error (text in hht_last_error) */
    HHT_ENCCL = 6,      /* NCCL error (text in hht_last_error) */
    HHT_EMISMATCH = 7,  /* ranks disagree on (N, depth, threshold, halves, images) */
    HHT_ESTATE = 8      /* getter called before a successful detect */
} hht_status;

#define HHT_ALPHA 1u    /* |m| <= 1 set: point (x, y) */
#define HHT_BETA 2u     /* |m| > 1 set: point taken as (y, x) */

#define HHT_EXACT 0u       /* opts.variant: the paper's exact corner-code test             */
#define HHT_FHT_CIRCLE 1u  /* opts.variant: FHT circumcircle test (comparison) */
#define HHT_FHT_CIRCLE_MB 2u  /* opts.variant: the same circle measured in (m, b) units (DESIGN R22) */

typedef struct hht_ctx hht_ctx;   /* opaque */
typedef struct hht_group hht_group;   /* opaque: in-process collective group (hht_group_create) */

typedef struct {
    int32_t device;          /* CUDA ordinal */
    int32_t rank;            /* this process's rank in [0, world) */
    int32_t world;           /* ranks sharing one detection (points sharded); 1 = single GPU */
    uint32_t halves;         /* HHT_ALPHA | HHT_BETA (default both) */
    uint32_t record_levels;  /* 1 (default): keep every level's (a, c, votes) records */
    uint32_t force_int64;    /* 1: use the int64 kernels even where int32 is exact (testing) */
    uint32_t profile;        /* 1: time every kernel launch with CUDA events (hht_result_profile) */
    uint32_t tail_depth;     /* dense leaf-grid tail: 0 = auto (5 when depth >= 5, else 4 when
                                depth >= 4, else 3); 6 (depth >= 6, exact test) = the fused tail
                                streams each level depth-5 region's parent list from level depth-6
                                (no level depth-5 or depth-4 lists); 5 = 16x16 grids of level
                                depth-4 rastered straight from level depth-5 lists (fused, no
                                level depth-4 lists);
                                4 = 16x16 grids from level depth-4 lists; 3 = 8x8 grids from level
                                depth-3 lists. Results are identical. */
    uint32_t prefetch;       /* pass/tail kernels: 0 = auto, 1 = fetch the next chunk's descriptor
                                only, 2 = also its list entries (more registers); 3 = list passes
                                fill a per-warp ring of two shared-memory slots with 1-D bulk copies
                                (cp.async.bulk + mbarrier) two chunks ahead; identical results */
    uint32_t latency_path;   /* 0 = auto: a small detection (one rank, exact test; bound on the
                                lists: sum over trees of points x (2^depth - 1) entries) runs as ONE
                                kernel launch: of one block (k_small) when all arrays fit 220 KiB of
                                shared memory, or (bound <= 2^16 entries) with the two lists in
                                device memory; else, for bounds up to 2^26 entries, as one
                                cooperative launch over the whole GPU (k_mid, stats.latency_path 2);
                                larger detections take the multi-kernel path. 1 = same as 0;
                                2 = never (always the multi-kernel path); 3 = k_mid whenever its
                                bounds admit the detection. Results are identical. The one-launch
                                paths also stage and range-check the points in that launch (an
                                out-of-range point still fails the call with HHT_ERANGE and no
                                results) and write the statistics to mapped host memory. */
    uint32_t variant;        /* membership test: HHT_EXACT (0, default) = the paper's 4-bit corner
                                code; HHT_FHT_CIRCLE (1) = the FHT comparison: the line meets the
                                region's circumscribing circle (exact integers, see
                                DESIGN.md). HHT_EOVERFLOW if 13 N^2 2^(2 depth - 1) >= 2^63;
                                HHT_FHT_CIRCLE_MB (2) = the same test with distance and radius in the
                                (m, b) units of the 2s/2^D x 3Ns/2^D rectangles (reading R22):
                                (2 G(centre))^2 <= (1 + ex^2)(4 + 9N^2) s^2, exact in 128 bits;
                                HHT_EOVERFLOW if (1 + N^2)(4 + 9N^2) 4^(depth-1) >= 2^126 */
    size_t mem_budget;       /* device bytes for candidate lists; 0 = 80% of free memory at create.
                                Levels whose lists do not fit are processed in depth-first ranges. */
    const void* nccl_id;     /* world > 1: 128-byte ncclUniqueId from hht_nccl_unique_id on rank 0,
                                identical on every rank. NULL when world == 1; a non-NULL id with
                                world == 1 runs every collective on a 1-rank communicator (tests) */
    hht_group* group;        /* instead of nccl_id: the ranks are `world` contexts of this process,
                                each driven by its own host thread, and every collective the
                                multi-rank path makes (the same calls, in the same order, as with
                                NCCL) is a host-staged allreduce among them. For testing the
                                multi-rank logic on one GPU; the contexts may share a device. */
    void* stream;            /* cudaStream_t the ctx enqueues all its work on, BORROWED (never
                                destroyed by the library); NULL: the ctx creates its own stream.
                                The legacy default stream is cudaStreamLegacy ((void*)1). Work the
                                caller enqueued on that stream before a detect call is ordered
                                before the detection (no host synchronisation needed). */
    void* nccl_comm;         /* ncclComm_t of `world` ranks, BORROWED (never destroyed by the
                                library); takes precedence over nccl_id; its size and rank must equal
                                world and rank (HHT_EINVAL otherwise) */
    uint32_t tail_units;     /* fused tail work units: 0 = auto (when a launch has fewer parents than
                                8 x its warps, each parent's chunks are split into blocks so every
                                warp has work to the end; with more parents, whole parents first and
                                then the last (one per warp) in pieces of 32 chunks, so that the launch
                                does not end waiting for the warps that took the last large parents);
                                2 = one unit per parent; 3 = always the second scheme (tests).
                                Identical results */
} hht_opts;

/* Re-point the ctx at another BORROWED stream (cudaStream_t; NULL = back to the ctx's own stream,
 * cudaStreamLegacy = (void*)1 for the legacy default stream) for the following calls. The previous
 * stream is synchronised first. Lets a caller order a detection after its own producer kernels on
 * its current stream without a host synchronisation (the Python binding passes torch's current
 * stream). */
hht_status hht_set_stream(hht_ctx* ctx, void* stream);

/* One detected line: leaf (i, j) of tree (image, half) with votes > threshold. */
typedef struct {
    int32_t image;
    uint32_t half;           /* HHT_ALPHA or HHT_BETA */
    uint32_t i, j;           /* leaf lattice indices (see conventions) */
    uint32_t votes;
} hht_leaf;

typedef struct {
    uint64_t tests;          /* line-region code evaluations: per tree E + 4 * sum of votes of every
                                split region (PAPER.md:296-298 unit; R9) */
    uint64_t votes;          /* sum of votes over every visited region (Table 1 "Number of votes") */
    uint64_t leaves;         /* detected lines */
    uint64_t pairs;          /* (split region, local candidate line) pairs streamed from HBM */
    uint64_t visited[64];    /* regions visited per level, all trees */
    uint64_t split[64];      /* regions split per level, all trees */
    uint64_t h2d_bytes, d2h_bytes;   /* host<->device bytes moved inside the call */
    uint32_t levels;         /* depth + 1 */
    uint32_t int_bits;       /* 32 or 64: corner arithmetic width used */
    uint32_t ranges;         /* list ranges processed (1 per level when everything fits) */
    uint32_t images;
    double ms;               /* device time of the call (CUDA events on the ctx stream) */
    uint64_t leaves_streamed;   /* leaf rows written to the leaf sink (hht_set_leaf_sink) */
    uint32_t latency_path;      /* 1: one-block latency path (k_small); 2: one cooperative launch
                                   (k_mid); 0: multi-kernel path */
    uint32_t reserved;
} hht_stats;

/* Leaf sink: while a detect runs, the detected lines are converted to hht_leaf rows and copied to
 * `host` as each leaf-level split finishes, on a second stream, overlapping the copies with the
 * rest of the traversal (depth-first ranges produce leaves in their final order). When the detect
 * returns, host[0 .. min(total, cap)) holds the same rows, in the same order, as
 * hht_result_leaves(ctx, -1, ...); stats.leaves is the total and stats.leaves_streamed the rows
 * written (fewer than the total only when cap is too small). `host` is borrowed until the sink is
 * replaced or removed (host = NULL); page-locked memory gives real overlap. */
hht_status hht_set_leaf_sink(hht_ctx* ctx, hht_leaf* host, int64_t cap);

/* Packed leaf sink: as hht_set_leaf_sink, but each detected line is one 8-byte row
 *     (uint64_t)i << 48 | (uint64_t)j << 32 | votes
 * (2.5x fewer bytes over PCIe than hht_leaf rows), in the same order (tree by tree: image order, ALPHA
 * before BETA, each tree in the paper's depth-first order); the tree of each row follows from
 * hht_result_tree_offsets. Replaces any row sink (and vice versa); host = NULL removes it. A detect
 * with depth > 16 and a packed sink set fails with HHT_EINVAL (i, j need 16 bits each). */
hht_status hht_set_leaf_sink_packed(hht_ctx* ctx, uint64_t* host, int64_t cap);

/* Leaf offsets per tree of the last detect: out[t] = index of tree t's first detected line in the
 * hht_result_leaves(ctx, -1, ...) / leaf-sink order, t = 0 .. ntrees (out[ntrees] = total), tree
 * t = image t / H, half index t % H (H = number of halves in opts.halves, ALPHA first). out holds
 * cap >= ntrees + 1 values; out = NULL: *ntrees only. */
hht_status hht_result_tree_offsets(hht_ctx* ctx, uint64_t* out, int64_t cap, int64_t* ntrees);

/* Per-kernel-class timings of the last detect (opts.profile = 1), CUDA events per launch. */
typedef struct {
    uint64_t launches[8];    /* 0 stage, 1 root count pass, 2 write pass (list compaction +
                                count-ahead), 3 dense tail (levels D-1, D) or count-only pass (D = 2),
                                4 split (threshold + scan), 5 chunk map / tail gather,
                                6 other (range selection), 7 allreduce */
    double ms[8];
    uint64_t bytes[8];       /* algorithmic HBM bytes moved by that class */
    uint64_t ops[8];         /* algorithmic integer instructions (thread-level) of that class where
                                it is issue-bound: the dense tail's raster steps; 0 else */
} hht_profile;

/* In-process collective group of `world` ranks (see hht_opts.group). Destroy after every context
 * that uses it. */
hht_status hht_group_create(hht_group** out, int32_t world);
void hht_group_destroy(hht_group* group);

/* Fill opts with defaults (device 0, rank 0 of 1, both halves, records on). */
hht_status hht_default_opts(hht_opts* opts);

/* Create a context on opts->device. For world > 1 this joins the NCCL communicator (collective:
 * every rank must call it). */
hht_status hht_create(hht_ctx** out, const hht_opts* opts);

/* Write a fresh 128-byte ncclUniqueId into out (cap >= 128). Call on rank 0 and broadcast. */
hht_status hht_nccl_unique_id(void* out, size_t cap);

/* Detect lines in one image: points = int32 [n][2] (x, y) with 0 <= x, y < N; depth D >= 1 is the
 * leaf level (PAPER.md:69 uses ceil(log2 N)); threshold T >= 1 (strict: votes > T splits / emits).
 * world > 1: each rank passes its own shard (n = local count); results are global and identical
 * on every rank. n = 0 is valid. */
hht_status hht_detect(hht_ctx* ctx, const int32_t* points, int64_t n, int32_t N, int32_t depth,
                      int64_t threshold);

/* Detect lines in B independent images at once (one tree per image and half): image b owns
 * points[offsets[b] .. offsets[b+1]) ; offsets is a HOST array of B+1 non-decreasing values with
 * offsets[0] = 0. */
hht_status hht_detect_batch(hht_ctx* ctx, const int32_t* points, const int64_t* offsets, int32_t B,
                            int32_t N, int32_t depth, int64_t threshold);

/* Detected lines of `image` (ALPHA tree first, each in the paper's depth-first NE,NW,SW,SE order);
 * image = -1 returns every image's lines in image order. */
/* solution() with point removal for the last detect: the
 * candidate leaves (hht_result_leaves) are taken in depth-first order within each tree and a leaf is
 * emitted iff more than `threshold` of its voters have not been removed by an earlier emitted leaf of
 * the same tree; its live voters are then removed (the paper's "exclude the edge point from further
 * calculations"). Rows (image, half, i, j, live votes), image -1 = all, same cap/count protocol as
 * hht_result_leaves. This equals the paper's depth-first detector with removal on (the oracle's
 * oracle_detect_removal). Computed on the GPU on first request and cached until the next detect, by
 * one cooperative kernel per group of trees: live vote counts per candidate, kept exact by rastering
 * each removed point's line over a dense 4^depth cell -> candidate map, so the next emission of every
 * tree is found in one scan (rounds <= points / threshold per tree). Device memory: 12 B per candidate
 * + 25 B per (tree, point) + 4^(depth+1) B per tree of a group (HHT_ENOMEM if one tree's map does not
 * fit the budget). Single rank, exact test only. */
hht_status hht_result_lines(hht_ctx* ctx, int32_t image, hht_leaf* out, int64_t cap, int64_t* count);

/* The supports of those lines: uint32 rows (line, point) sorted by line then point, where line indexes
 * the rows hht_result_lines returns for the same `image` (-1: all images, global line index) and point
 * indexes the point set of the line's tree (the image's points for hht_detect / hht_detect_batch; the
 * tree's own set for hht_detect_trees). Every point appears at most once per tree (it is removed by the
 * line it supports). out holds cap rows (2 * cap uint32); out = NULL: count only. */
hht_status hht_result_line_points(hht_ctx* ctx, int32_t image, uint32_t* out, int64_t cap, int64_t* count);

/* Per-tree point sets (each point in ONE tree, e.g. the edge front end's ALPHA/BETA partition,
 * PAPER.md:67): tree t = image t / H + half index t % H (H = number of halves in opts.halves,
 * ALPHA first) gets the int2 (x, y) points [tree_offsets[t], tree_offsets[t+1]) of `points`
 * (device or host, same conventions as hht_detect_batch); tree_offsets is host int64 [B*H + 1].
 * Results are read with the same getters. Multi-rank: each rank passes its local points per tree. */
hht_status hht_detect_trees(hht_ctx* ctx, const int32_t* points, const int64_t* tree_offsets, int32_t B,
                            int32_t N, int32_t depth, int64_t threshold);

/* Edge front end + detection of one square grayscale image (readings
 * DESIGN.md R18-R21 after SPEC.md:104-131): img is uint8 [N][N] row-major, row 0 = top (device or
 * host). Interior pixels get the 3x3 Sobel gradient in geometric coordinates (x = column,
 * y = N-1-row); a pixel is an edge point iff |gx| + |gy| >= mag_threshold > 0; it goes to ALPHA iff
 * |gx| <= |gy|, else to BETA; then the ALPHA tree is run on the ALPHA points and the BETA tree on
 * the BETA points (hht_detect_trees). 3 <= N <= 46340; one rank only. */
hht_status hht_detect_image(hht_ctx* ctx, const uint8_t* img, int32_t N, int32_t mag_threshold, int32_t depth,
                            int64_t threshold);

/* The edge points of the last hht_detect_image as host int2 (x, y): the ALPHA set then the BETA set
 * (only the halves in opts.halves), each in raster order. out = NULL: counts only. Invalidated by
 * the next detect call. HHT_EINVAL if cap < n_alpha + n_beta; HHT_ESTATE without such a result. */
hht_status hht_result_edges(hht_ctx* ctx, int32_t* out, int64_t cap, int64_t* n_alpha, int64_t* n_beta);

hht_status hht_result_leaves(hht_ctx* ctx, int32_t image, hht_leaf* out, int64_t cap, int64_t* count);

/* Visited regions of tree (image, half) at `level` in depth-first quad order, as uint32 triplets
 * (a, c, votes): out holds cap triplets (3*cap uint32). Needs opts.record_levels = 1. */
hht_status hht_result_level(hht_ctx* ctx, int32_t image, uint32_t half, int32_t level, uint32_t* out,
                            int64_t cap, int64_t* count);

hht_status hht_result_stats(hht_ctx* ctx, hht_stats* out);
hht_status hht_result_profile(hht_ctx* ctx, hht_profile* out);

/* One kernel launch of the last detect (opts.profile = 1), in launch order. */
typedef struct {
    uint32_t cls;            /* hht_profile class index */
    uint32_t reserved;
    uint64_t bytes;          /* algorithmic HBM bytes of this launch */
    double ms;               /* CUDA-event duration */
} hht_launch;

/* Per-launch log of the last detect (opts.profile = 1); same cap/count protocol as the getters. */
hht_status hht_result_launches(hht_ctx* ctx, hht_launch* out, int64_t cap, int64_t* count);

/* Device-time bracket on the ctx stream (CUDA events): begin records, end records, synchronises
 * and returns the milliseconds between the two. */
hht_status hht_timer_begin(hht_ctx* ctx);
hht_status hht_timer_end(hht_ctx* ctx, double* ms);

/* One line describing the last error of ctx (never NULL; "" if none). */
const char* hht_last_error(const hht_ctx* ctx);
const char* hht_status_str(hht_status s);

/* Release every resource; NULL-safe; synchronises the ctx stream first. */
void hht_destroy(hht_ctx* ctx);

/* Library build identification: "hht <version> sm_100a build <id>", id = 16 hex digits of the sha256
 * of the CUDA sources, headers and nvcc flags it was built from (equal for every build of the same
 * kernels, unlike the bytes of the .so). */
const char* hht_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HHT_H */

/*
 * spectree_b200 -- C ABI of the B200-native classification-tree evaluator.
 *
 * This is the drop-in boundary for the reference's evaluate API
 * (/root/reference/proj/core).  Every entry point is plain C: pointers, sizes
 * and POD structs, no C++ or torch types.  The reference-side binding a
 * maintainer adds is in INTEGRATION.md; the C++ wrapper that mirrors the
 * reference signatures exactly is include/spectree_b200.hpp.
 *
 * Semantics are the reference's, bit for bit:
 *   successor(i, x) = child(i) + (uint32)(x[attr(i)] > thr(i))    tree.hpp:51-54
 *   walk from node 0 until class_id != ST_NO_CLASS                 eval_serial.cpp:21-29
 *   one uint32 label per record, positional                        dataset.hpp:35-36
 * (ordered IEEE '>' without flush-to-zero: ties and NaN go left.)
 *
 * Return codes mirror the reference error taxonomy / CLI exit codes
 * (errors.hpp:12-46, main.cpp:703-712):
 *   0 ok, 2 argument (ArgumentError), 3 io/parse, 4 CUDA failure,
 *   5 no CUDA device.  There is NO CPU fallback: without a usable device
 *   every evaluating call returns 5.
 * st_last_error() returns the thread-local message of the last failure.
 *
 * Thread safety: trees/forests are immutable after creation and may be shared
 * by concurrent callers (device replicas are created lazily under a lock),
 * like the reference's pure evaluators.
 */
#ifndef SPECTREE_B200_H
#define SPECTREE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ST_NO_CLASS 0xFFFFFFFFu /* spectree::kNoClass, tree.hpp:15-16 */

/* Layout-identical to spectree::EncodedNode (tree.hpp:43-55), 16 bytes:
 * {u32 attribute @0, f32 threshold @4, u32 child @8, u32 class_id @12}. */
typedef struct st_node {
  uint32_t attribute;
  float threshold;
  uint32_t child;
  uint32_t class_id;
} st_node;

enum st_status {
  ST_OK = 0,
  ST_ERR_ARGUMENT = 2,
  ST_ERR_IO = 3,
  ST_ERR_CUDA = 4,
  ST_ERR_NO_DEVICE = 5
};

/* Feature matrix layout.  AoS = the reference Dataset (row-major, record(i) =
 * values + i*ld, dataset.hpp:20-22).  SoA = attribute-major, x[a*ld + r]. */
enum st_layout { ST_LAYOUT_AOS = 0, ST_LAYOUT_SOA = 1 };

/* Algorithm 1 = data decomposition (eval_data_parallel.cpp:35-88),
 * Algorithm 2 = speculative decomposition (eval_speculative.cpp:207-273). */
enum st_algo { ST_ALGO_AUTO = 0, ST_ALGO_DATA = 1, ST_ALGO_SPECULATIVE = 2 };

/* Where the data kernel reads the node array from. */
enum st_tree_loc {
  ST_TREE_AUTO = 0,
  ST_TREE_SHARED = 1,   /* staged once per CTA into shared memory */
  ST_TREE_CONSTANT = 2, /* __grid_constant__ kernel parameter (constant bank), N <= 4000 */
  ST_TREE_GLOBAL = 3    /* read-only global path (L1/L2), any size */
};

/* GPU geometry.  Zero-initialise for defaults (st_geom_default). */
typedef struct st_geom {
  uint32_t algo;               /* st_algo */
  uint32_t tree_loc;           /* st_tree_loc (data kernel) */
  uint32_t samples_per_thread; /* data kernel: independent walks per lane (0 = auto);
                                  speculative ring: record streams per group, 1 or 2 (0 = auto) */
  uint32_t group_lanes;        /* speculative: lanes per record group, power of two <= 32 (0 = auto) */
  uint32_t window_levels;      /* speculative: max window height in tree levels (0 = auto) */
  uint32_t reductions;         /* speculative: 0 = fixed per-window doubling count;
                                  k >= 1 = check the root after every k doublings
                                  (reference ReductionMode::barrier_separated, k = reductions_per_iteration) */
  uint32_t blocks_per_sm;      /* 0 = occupancy-derived persistent grid */
  uint32_t stages;             /* TMA record-pipeline stages per warp (0 = auto, 1-8) */
  uint32_t warps_per_cta;      /* CTA width in warps, 1-32 (0 = auto) */
  uint32_t pipeline;           /* speculative record staging: 0 = auto (CTA-shared ticketed TMA
                                  ring), 1 = per-warp TMA ring */
  uint32_t record_regs;        /* data kernel, 8/16-attribute records: 0 = auto (transposed tile for 8),
                                  1 = walk from registers (tile released right after loading),
                                  2 = walk from the shared tile,
                                  3 = transpose each tile in place to attribute-major, then walk it */
  uint32_t variant;            /* ST_VAR_* bit flags: A/B variants of the tuned defaults (0 = defaults) */
  uint32_t ring_slots;         /* speculative ring: cap on the tile-slot count (0 = auto; stress tests) */
  uint32_t slot_records;       /* speculative ring: records per slot / 32, 1 or 2 (0 = auto); with lane
                                  triples 2 = 80-record and 3 = 120-record slots */
  uint32_t fold_min;           /* data kernel: fold trees of at least this many nodes (0 = auto: 2047) */
  uint32_t pdl;                /* data kernel: programmatic dependent launch, 0 = auto,
                                  1 = trigger dependents early, 2 = at exit, 3 = off */
  uint32_t forest_chains;      /* forest: trees walked per lane at once, 1-4 (0 = auto) */
  uint32_t forest_slots;       /* forest: shared-memory tree ring slots (0 = auto) */
  uint32_t reserved[6];
} st_geom;

/* st_geom.variant flags.  Every combination gives identical labels; they
 * select the implementation variants the tuned defaults were measured
 * against, so tests and A/B tools reach them per call. */
enum st_variant {
  ST_VAR_NO_FOLD = 1u,      /* data / forest: never fold leaf pairs into terminal nodes */
  ST_VAR_TREE_LOOP = 2u,    /* stage trees / window tables with per-thread loads, not one bulk copy */
  ST_VAR_SPEC_GENERAL = 4u, /* speculative, one-window trees: the general window loop */
  ST_VAR_SPEC_JUMP = 8u,    /* speculative, one-window trees: shfl pointer jumping instead of
                               the ballot + leaf path-mask reduction */
  ST_VAR_SPEC_WIDE = 16u,   /* speculative: 16-byte window entries instead of 8-byte ones */
  ST_VAR_SPEC_SELECT = 32u, /* speculative: a select per pointer-jumping step (round-1 codes) instead
                               of self-loop terminal codes */
  ST_VAR_SPEC_PRED = 64u,   /* speculative, self-loop two-stream loop: predicated stream advance */
  ST_VAR_SPEC_BRANCH = 128u,/* ... the stream advance in a divergent branch (default: by tree shape) */
  ST_VAR_SPEC_FIXED = 256u, /* ... every record runs the deepest window count, leaves absorbing */
  ST_VAR_SPEC_QUAD = 512u   /* ... fixed-trip loop on 4-lane groups (8 records per warp step) instead of
                               interleaved lane triples (10) */
};

/* Optional per-record speculative counters (SpeculativeStats,
 * eval_speculative.hpp:73-77).  Arrays of m uint32, in the same memory space
 * as the labels of the call they are passed to. */
typedef struct st_stats {
  uint32_t* iterations;     /* reduction-loop trips (summed over windows) */
  uint32_t* doubling_steps; /* pointer-jumping steps applied */
} st_stats;

typedef struct st_tree_info {
  uint32_t nodes, leaves, internal, depth, max_attribute;
  uint32_t compact;        /* 1 if the 8-byte device node format applies */
  uint32_t spec_windows;   /* speculative windows for the default geometry */
  uint32_t spec_group_lanes;
  uint32_t max_class;      /* largest leaf class id (u8 label files need < 256) */
} st_tree_info;

typedef struct st_tree st_tree;
typedef struct st_forest st_forest;

const char* st_last_error(void);
const char* st_version(void);
int st_device_count(int* count);
void st_geom_default(st_geom* g);

/* Tree-load boundary: replaces constructing spectree::EncodedTree for the GPU
 * (tree.hpp:61-92, EncodedTree ctor tree.cpp:35-61).  Rejects, with
 * ST_ERR_ARGUMENT, n == 0 and any internal node whose child link is not
 * strictly forward or whose right child is out of range (the subset of
 * validate(), tree.cpp:138-189, that a walk needs to terminate in bounds). */
int st_tree_create(const st_node* nodes, uint32_t n, st_tree** out);
void st_tree_destroy(st_tree* tree);
int st_tree_get_info(const st_tree* tree, st_tree_info* out);

/* Random forest: t trees, per-sample majority vote over their labels, smallest
 * class id on ties.  Every leaf class must be < n_classes (<= 64). */
int st_forest_create(const st_node* const* trees, const uint32_t* sizes, uint32_t t,
                     uint32_t n_classes, st_forest** out);
void st_forest_destroy(st_forest* forest);

/* Host-buffer evaluation ("outer" window of bench.cpp:267-296): copies the
 * records in, runs the kernel on the current CUDA device, copies labels out;
 * chunked and pipelined over three streams (H2D of chunk c+1 beside the
 * kernel and D2H of chunk c).  x is m records of arity a
 * (AoS: ld >= a floats between records; SoA: ld >= m floats between
 * attributes; ld = 0 means packed).  labels: m uint32.  Throws the
 * reference's ArgumentError (code 2) before any work when
 * max_attribute >= a (check_attribute_range, eval_serial.cpp:10-17).
 * m == 0 returns immediately with no launch. */
int st_eval(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld,
            int layout, const st_geom* geom, uint32_t* labels, st_stats* stats);

/* Device-resident evaluation ("inner" window): x and labels are device
 * pointers on the current device, enqueued on `stream` (a cudaStream_t, NULL =
 * legacy default stream).  Asynchronous: no host synchronisation. */
int st_eval_device(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                   int layout, const st_geom* geom, uint32_t* labels, st_stats* stats,
                   void* stream);

/* Sample-sharded evaluation over several devices of one box: device k owns
 * records [floor(k*m/n), floor((k+1)*m/n)) (the Proc. 3 range rule,
 * eval_data_parallel.cpp:47-51); the tree is replicated, labels are gathered
 * into disjoint slices of `labels`.  No collective in the hot loop. */
int st_eval_sharded(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                    int layout, const st_geom* geom, const int* devices, int ndev,
                    uint32_t* labels);

/* Forest evaluation: host buffers (st_forest_eval, same pipeline as st_eval)
 * or device pointers on `stream`.  geom (nullable) carries warps_per_cta,
 * forest_chains, forest_slots and ST_VAR_NO_FOLD; other fields are ignored. */
int st_forest_eval(const st_forest* forest, const float* x, uint64_t m, uint32_t a,
                   uint64_t ld, int layout, const st_geom* geom, uint32_t* labels);
int st_forest_eval_device(const st_forest* forest, const float* x, uint64_t m, uint32_t a,
                          uint64_t ld, int layout, const st_geom* geom, uint32_t* labels,
                          void* stream);

/* Traversal depths (reference traversal_depths, eval_serial.cpp:77-105): per
 * record, the number of edges from the root to the leaf it reaches, written
 * by the data-decomposition kernel beside the labels (one pass over the
 * records).  st_eval_depths takes host buffers (same pipeline as st_eval);
 * st_eval_depths_device device pointers on `stream`.  labels and depths: m
 * uint32 each.  The reference's mean_traversal_depth (:99-110) is the mean of
 * `depths` (the C++ / Python mirrors throw ArgumentError on an empty
 * dataset, as the reference does).  geom->algo is ignored (always data). */
int st_eval_depths(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                   int layout, const st_geom* geom, uint32_t* labels, uint32_t* depths);
int st_eval_depths_device(const st_tree* tree, const float* x, uint64_t m, uint32_t a,
                          uint64_t ld, int layout, const st_geom* geom, uint32_t* labels,
                          uint32_t* depths, void* stream);

/* ---- resident frame stream (C3: video-rate per-pixel classification) ----
 * One grid stays resident -- the data decomposition, or with geom->algo =
 * ST_ALGO_SPECULATIVE the speculative ring's fixed-trip window loop (trees
 * with > 32 internal nodes, records a multiple of its 32 / 80 / 120-record
 * slots) -- and classifies frame 0, 1, 2,
 * ... as they are published into a device ring of `ring` frame slots of
 * `records` records x `a` attributes (AoS float32; a = 8, 16 or 32; records a
 * multiple of the walk's tile, 32..128 records): the tree is staged once, no
 * launch per frame.  Frame seq lives in slot seq % ring (st_frames_slot gives
 * its device pointers).  Stream-ordered protocol for device producers:
 *   st_frames_acquire(seq, s)  s waits until frame seq - ring is done (slot free)
 *   ... producer work on s writes the slot's records ...
 *   st_frames_publish(seq, s)  after s's prior work, frames up to seq are ready
 *   st_frames_wait(seq, s2)    s2 waits until frame seq's labels are written
 * Frames complete in order, so one acquire of the last frame of a batch
 * (seq + k) frees the slots of frames seq .. seq + k, and one publish of it
 * publishes the batch; a frame must be acquired before it is published.
 * (cuStreamWriteValue32 / cuStreamWaitValue64: no SM time).  Host convenience:
 * st_frames_push copies host records into the next slot and publishes them;
 * st_frames_pop waits for a frame and copies its labels out (pop frame seq
 * before publishing frame seq + ring).  The resident grid owns the SMs it
 * occupies (max_ctas caps it, 0 = the planned persistent grid); device-wide
 * synchronisation (cudaDeviceSynchronize, cudaFree) waits for it until
 * st_frames_close.  A grid idle for idle_timeout_ms (0 = 10 s) stops itself
 * (st_frames_status reports it).  Labels equal st_eval's for every frame. */
typedef struct st_frames st_frames;
int st_frames_open(const st_tree* tree, uint64_t records, uint32_t a, uint32_t ring, const st_geom* geom,
                   uint32_t max_ctas, uint32_t idle_timeout_ms, st_frames** out);
int st_frames_slot(st_frames* f, uint64_t seq, float** records, uint32_t** labels);
int st_frames_acquire(st_frames* f, uint64_t seq, void* stream);
int st_frames_publish(st_frames* f, uint64_t seq, void* stream);
int st_frames_wait(st_frames* f, uint64_t seq, void* stream);
int st_frames_push(st_frames* f, const float* host_records, uint64_t* seq);
int st_frames_pop(st_frames* f, uint64_t seq, uint32_t* host_labels);
int st_frames_status(st_frames* f, uint64_t* published, uint32_t* stopped);
int st_frames_close(st_frames* f);

/* One unpipelined host round trip with per-phase timing: the GPU edition of
 * the reference bench windows (bench.hpp:50-56, bench.cpp:228-262) and of the
 * paper's Table 1 (allocation, copy-in, kernel, copy-out, release):
 *   outer_us = the whole call on the host steady clock (alloc + H2D + kernel
 *              + D2H + free), the reference's "outer" window
 *   inner_us = the evaluation kernel(s) only (CUDA events), the "inner" window
 *   alloc_us = device buffer cudaMalloc + cudaFree (host clock), "alloc"
 *   h2d_us / d2h_us = the record and label copies (CUDA events)
 * Same arguments, validation and labels as st_eval (stats not supported). */
typedef struct st_timing {
  double outer_us, inner_us, alloc_us, h2d_us, d2h_us;
} st_timing;
int st_eval_timed(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                  int layout, const st_geom* geom, uint32_t* labels, st_timing* timing);

/* ---- record and label files at scale ------------------
 * The reference's CSV loader (io.cpp:80-117) is parse-bound; this is a raw
 * little-endian float32 format that streams at disk / PCIe speed.
 *
 * Record file: 64-byte header, then count*arity float32 (AoS: record-major,
 * SoA: attribute-major).
 *   @0 char[8] "STREC001"   @8 u32 version = 1   @12 u32 layout (st_layout)
 *   @16 u64 count           @24 u32 arity (>= 1, dataset.cpp:10-14)
 *   @28 u32 flags (bit 0: checksum present)      @32 u64 checksum
 *   @40..63 zero
 * checksum = dataset_checksum (dataset.cpp:76-93) of the records in record
 * order, so a file round-trips to the reference's own checksum.
 * Label file: 32-byte header, then count labels of `width` bytes (4 = u32,
 * 1 = u8 when every class < 256).
 *   @0 char[8] "STLAB001"   @8 u32 version = 1   @12 u32 width (1 | 4)
 *   @16 u64 count           @24..31 zero
 * Malformed headers / short files return ST_ERR_IO (the reference's
 * IoError / ParseError exit code 3). */
typedef struct st_dataset_info {
  uint64_t count;
  uint32_t arity;
  uint32_t layout;
  uint32_t has_checksum;
  uint64_t checksum;
  uint64_t data_offset; /* byte offset of the first value */
} st_dataset_info;

int st_dataset_save(const char* path, const float* x, uint64_t m, uint32_t a, int layout,
                    int with_checksum);
int st_dataset_info_read(const char* path, st_dataset_info* out);
/* Reads records [first, first+count) into `out` (count*arity floats, AoS,
 * whatever the file layout).  verify != 0 re-computes the header checksum
 * over the whole file first (ST_ERR_IO on mismatch). */
int st_dataset_load(const char* path, uint64_t first, uint64_t count, float* out, int verify);
int st_labels_save(const char* path, const uint32_t* labels, uint64_t m, uint32_t width);
/* count of labels in the file (and width); out may be NULL to size. */
int st_labels_load(const char* path, uint32_t* out, uint64_t cap, uint64_t* count, uint32_t* width);

/* Streams a record file through the GPU: a reader thread fills pinned
 * buffers with ~64 MB chunks while the previous chunks are copied in,
 * evaluated (st_eval_device) and their labels copied out and appended to
 * `labels_path` (width 1 narrows to u8 on the device; ST_ERR_ARGUMENT when a
 * leaf class is >= 256).  The whole file never has to fit in host memory
 * (C5: 10^9 records = 64 GB).  *records_out (nullable) = records classified. */
int st_eval_file(const st_tree* tree, const char* data_path, const st_geom* geom,
                 const char* labels_path, uint32_t width, uint64_t* records_out);

/* Number of kernel launches the last successful evaluating call on this
 * thread enqueued (for bench.py's gpu_launches claim). */
uint32_t st_last_launch_count(void);

/* ---- input side of the boundary (reference layer L1) ----------------------
 * Canonical synthetic inputs, bit-identical to the reference generators for
 * the same seed: generate_synthetic_tree (synthetic.cpp:82-154, breadth-first
 * encoded as by encode_breadth_first, tree.cpp:72-113) and
 * generate_synthetic_dataset (synthetic.cpp:156-182; gaussian != 0 selects
 * Distribution::gaussian).  st_synthetic_tree writes at most `cap` nodes and
 * always sets *n_out to the node count (call with out = NULL to size).
 * Infeasible shapes return ST_ERR_ARGUMENT with the reference's message. */
int st_synthetic_tree(uint32_t depth, uint32_t leaves, uint32_t arity, uint32_t classes,
                      uint64_t seed, st_node* out, uint32_t cap, uint32_t* n_out);
int st_synthetic_dataset(uint64_t count, uint32_t arity, uint64_t seed, int gaussian, float* out);
/* dataset_checksum (dataset.cpp:76-93) and raw FNV-1a-64 (label hashes). */
uint64_t st_dataset_checksum(const float* x, uint64_t count, uint32_t arity);
uint64_t st_fnv1a64(const void* data, uint64_t n);

#ifdef __cplusplus
}
#endif

#endif /* SPECTREE_B200_H */

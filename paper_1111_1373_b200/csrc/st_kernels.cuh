// sm_100a device code for the classification-tree hot path.
//
//   k_data   -- Algorithm 1, data decomposition (paper Proc. 3, PAPER.md:423-447;
//               reference eval_data_parallel.cpp:47-60): one lane walks S records.
//   k_spec   -- Algorithm 2, speculative decomposition (paper Procs. 4/5,
//               PAPER.md:537-647; reference eval_speculative.cpp:127-204): a group
//               of G lanes evaluates every internal node of a window in parallel
//               and resolves the path by shfl pointer-jumping.
//   k_forest -- T trees per record with a per-record majority vote.
//
// Record staging (shared by all three): every warp owns a private ring of NS
// shared-memory stages.  Lane 0 streams whole tiles of 32*S records from HBM
// with TMA (cp.async.bulk.tensor.2d over the record matrix viewed as rows of
// 32 floats, SWIZZLE_128B) completing on a per-stage mbarrier; the warp walks
// stage i while stages i+1..i+NS-1 are in flight.  No registers hold
// prefetched data and no instructions are spent on staging.  The 128B swizzle
// spreads "all lanes read the same attribute of 32 records" (every root
// visit) over 8 bank groups.  Non-TMA inputs (strided rows, SoA, unaligned
// base, the partial last tile) are stored by the warp into the same swizzled
// layout, so the walk code is identical.
//
// Semantics (bit-exact with the reference): successor = child + (x > thr)
// with an ordered IEEE compare and no flush-to-zero (tree.hpp:51-54); build
// without --use_fast_math / -ftz=true.
#pragma once
#include <cuda.h>  // CUtensorMap (type only; encoded on the host via the runtime entry point)
#include <cuda_runtime.h>

#include <cstdint>

namespace stk {

constexpr uint32_t kLeafBit = 0x80000000u;  // compact-node meta: leaf marker
constexpr uint32_t kExitBit = 0x40000000u;  // speculative code: exit to window
// Folded data-walk trees: a node whose two children are both leaves becomes a
// terminal  {thr, kLeafBit | kPairBit | classR << 20 | classL << 10 | 4*attr}
// (classes < 1024, 4*attr < 1024); its leaf pair is dropped from the array.
constexpr uint32_t kPairBit = 0x40000000u;
constexpr uint32_t kNoClass = 0xFFFFFFFFu;
constexpr int kWarpsPerCta = 8;    // default CTA width (warps); launches may use up to 32
constexpr int kMaxThreads = 1024;
constexpr int kForestMaxThreads = 768;  // k_forest_smem: <= 24 warps (the tile ring fits ~21): up to 80 registers
constexpr int kTripleSlot = 80;   // records per ring slot of the lane-triple speculative loop (x 3/2: L3 = 3)

// Compact 8-byte device node.  internal: meta = (8*child) << abits | 4*attr
// (bit 31 clear; byte offsets so the walk does no scaling); leaf: meta =
// kLeafBit | class (or | leaf ordinal when a class does not fit in 31 bits;
// the host then passes a leaf-class table).
struct __align__(8) CNode {
  float thr;
  uint32_t meta;
};

// Speculative window entry (16 B): lane j of a window evaluates one internal
// node.  attr_steps = 4*attr | steps << 24 (steps = doubling count that
// resolves this window); left/right = successor codes: < 32 lane index inside
// the window, kExitBit | base of the next window, kLeafBit | class/ordinal.
struct __align__(16) SEntry {
  float thr;
  uint32_t attr_steps;
  uint32_t left;
  uint32_t right;
};

enum Loader { kTma = 0, kScalar = 1, kSoa = 2, kDirect = 3 };
// kSharedReg: shared-memory tree, records walked from registers (8-attribute
// records; the TMA tile is released as soon as it is in registers).
// kSharedT: shared-memory tree, each warp's tile transposed in place to
// attribute-major (feature reads conflict-free, no register select); the
// staged tree's attribute fields are pre-scaled to the transposed stride.
enum TreeLoc { kShared = 1, kConst = 2, kGlobal = 3, kWide = 4, kSharedReg = 5, kSharedT = 6 };

// ---------------------------------------------------------------------------
// PTX helpers (32-bit shared addresses)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_u2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds_u4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// 1-D bulk copy global -> shared completing on an mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// Byte offset of flat float f of a tile under SWIZZLE_128B (tile base
// 1024-aligned): 16-byte chunk bits [4:6] XOR row bits [7:9].
__device__ __forceinline__ uint32_t swz(uint32_t byte_off) {
  return byte_off ^ ((byte_off >> 3) & 0x70u);
}

// Low halves of two codes in one word (PRMT): self-loop codes are < 2^16
// (WinTable::sl_cbits <= 15), so one root broadcast serves two record
// streams -- a shuffle costs ~1.8 shared-pipe cycles per warp instruction
// (profiles/r2_mio_probe.txt), two integer ops cost none of it.
__device__ __forceinline__ uint32_t pack_lo16(uint32_t lo, uint32_t hi) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, 0x5410;" : "=r"(r) : "r"(lo), "r"(hi));
  return r;
}

// ---------------------------------------------------------------------------
// Per-record feature accessor over a staged tile (or global for kDirect).
// get(attr4) takes the attribute as a byte offset (4 * attribute).
// ---------------------------------------------------------------------------
template <int A, int LOADER>
struct Rec {
  static constexpr bool kRowLocal = A > 0 && A <= 32 && (32 % A) == 0;  // record inside one 128 B row
  uint32_t base, xm;
  const float* gp;   // kDirect: the record's first feature
  uint32_t astride;  // kDirect: floats between consecutive attributes (1 AoS, ld SoA)

  // `ld` is the layout's leading dimension; soa selects x[a*ld + row].
  __device__ __forceinline__ void init(uint32_t tile, uint32_t r, uint32_t a_rt, const float* x,
                                       uint64_t row, uint32_t ld, uint32_t soa = 0) {
    if constexpr (LOADER == kDirect) {
      gp = soa ? x + row : x + row * (uint64_t)ld;
      astride = soa ? ld : 1u;
    } else if constexpr (kRowLocal) {
      const uint32_t ra4 = r * (uint32_t)A * 4u;
      const uint32_t rowb = ra4 & ~127u;
      base = tile + rowb;
      xm = ((rowb >> 3) & 0x70u) ^ (ra4 & 127u);
    } else {
      base = tile + r * (A > 0 ? (uint32_t)A : a_rt) * 4u;
    }
  }
  // Move to record r_new of the same tile, dr records further on.
  __device__ __forceinline__ void advance(uint32_t r_new, uint32_t dr, uint32_t a_rt, uint32_t tile,
                                          const float* x, uint64_t row_new, uint32_t ld,
                                          uint32_t soa) {
    if constexpr (LOADER == kDirect) {
      init(tile, r_new, a_rt, x, row_new, ld, soa);
    } else if constexpr (kRowLocal) {
      if constexpr ((A * 4) % 128 == 0) {
        // whole rows per record: base moves by dr rows; xm only depends on r & 7
        base += dr * (uint32_t)A * 4u;
        xm = (((r_new * (uint32_t)A * 4u) >> 3) & 0x70u);
      } else {
        init(tile, r_new, a_rt, x, row_new, ld, soa);
      }
    } else {
      base += dr * (A > 0 ? (uint32_t)A : a_rt) * 4u;
    }
  }
  __device__ __forceinline__ float get(uint32_t attr4) const {
    if constexpr (LOADER == kDirect) {
      return __ldg(gp + (uint64_t)(attr4 >> 2) * astride);
    } else if constexpr (kRowLocal) {
      return lds_f32(base + (attr4 ^ xm));
    } else {
      const uint32_t f = base + attr4;
      return lds_f32(f ^ ((f >> 3) & 0x70u));
    }
  }
};

// ---------------------------------------------------------------------------
// Per-warp record pipeline.  Tile t covers records [t*R, t*R + R), R = 32*S.
// ---------------------------------------------------------------------------
struct PipeArgs {
  const float* x;
  uint64_t m;
  uint32_t a, ld;
  uint32_t layout_soa;
};

template <int A, int S, int LOADER>
struct Pipe {
  static constexpr int R = 32 * S;
  uint32_t tiles, bars, stride_bytes, ns;
  const CUtensorMap* tmap;
  PipeArgs p;
  int lane;
  uint32_t row0 = 0;  // first 128-byte row of the record range in the tensor map (frame slot)

  __device__ __forceinline__ uint32_t arity() const { return A > 0 ? (uint32_t)A : p.a; }
  __device__ __forceinline__ bool full(uint64_t t) const { return (t + 1) * (uint64_t)R <= p.m; }
  __device__ __forceinline__ uint32_t stage(uint32_t s) const { return tiles + s * stride_bytes; }

  __device__ __forceinline__ void issue(uint64_t t, uint32_t s) {  // lane 0
    const uint32_t bytes = R * arity() * 4u;
    const uint32_t bar = bars + 8u * s;
    mbar_arrive_expect_tx(bar, bytes);
    tma_load_2d(stage(s), tmap, 0, (int)(row0 + t * (uint64_t)R * arity() / 32u), bar);
  }

  __device__ __forceinline__ void start(uint64_t first, uint64_t step, uint64_t n_tiles) {
    if constexpr (LOADER == kTma) {
      if (lane == 0) {
        tma_prefetch_desc(tmap);
        for (uint32_t s = 0; s < ns; ++s) mbar_init(bars + 8u * s, 1);
        fence_barrier_init();
        for (uint32_t s = 0; s < ns; ++s) {
          const uint64_t t = first + s * step;
          if (t < n_tiles && full(t)) issue(t, s);
        }
      }
      __syncwarp();
    }
  }

  // Make this warp's i-th tile (global index t) resident; returns its stage.
  __device__ __forceinline__ uint32_t acquire(uint64_t i, uint64_t t) {
    if constexpr (LOADER == kDirect) return 0;
    const uint32_t s = (uint32_t)(i % ns);
    const uint32_t dst = stage(s);
    if constexpr (LOADER == kTma) {
      if (full(t)) {
        mbar_wait(bars + 8u * s, (uint32_t)((i / ns) & 1u));
        return dst;
      }
    }
    // warp-cooperative store into the swizzled layout (scalar / SoA / tail)
    const uint32_t a = arity();
    const uint64_t r0 = t * (uint64_t)R;
    const uint32_t rows = (uint32_t)((p.m - r0) < (uint64_t)R ? (p.m - r0) : (uint64_t)R);
    __syncwarp();
    if (p.layout_soa) {
      for (uint32_t aa = 0; aa < a; ++aa)
        for (uint32_t r = lane; r < R; r += 32)
          sts_f32(dst + swz((r * a + aa) * 4u),
                  r < rows ? __ldg(p.x + (uint64_t)aa * p.ld + r0 + r) : 0.0f);
    } else {
      const uint32_t total = rows * a;
      for (uint32_t f = lane; f < total; f += 32) {
        const uint32_t r = f / a, aa = f - r * a;
        sts_f32(dst + swz(f * 4u), __ldg(p.x + (r0 + r) * (uint64_t)p.ld + aa));
      }
    }
    __syncwarp();
    return dst;
  }

  // Done with this warp's i-th tile: refill its stage with tile t + ns*step.
  // Every lane's generic-proxy accesses to the stage (reads; the transposed
  // walk's stores) are ordered before lane 0's async-proxy TMA write by a
  // proxy fence on each lane, then the warp barrier.
  __device__ __forceinline__ void release(uint64_t i, uint64_t t, uint64_t step, uint64_t n_tiles) {
    if constexpr (LOADER == kTma) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if constexpr (LOADER == kTma) {
      if (lane == 0) {
        const uint64_t tn = t + ns * step;
        if (tn < n_tiles && full(tn)) issue(tn, (uint32_t)(i % ns));
      }
    }
  }
};

// ---------------------------------------------------------------------------
// Tree access (byte offsets: root at 0, child at meta >> abits)
// ---------------------------------------------------------------------------
template <int CAP>
struct ConstTree {
  CNode n[CAP];
};

// Shared-memory trees are rebased when staged: an internal node's child field
// then holds the child's absolute shared-memory byte address, so the walk's
// next-node address is (meta >> abits) + 8*(x > thr) with no base add.
// Constant / global trees keep offsets relative to node 0.
template <int TLOC>
constexpr bool kAbsTree = (TLOC == kShared || TLOC == kSharedReg || TLOC == kSharedT);

template <int TLOC, int CAP>
struct TreeRef {
  uint32_t s;                   // shared address of node 0
  const char* g;                // global node array
  const ConstTree<CAP>* c;      // constant-bank copy
  __device__ __forceinline__ uint32_t root() const { return kAbsTree<TLOC> ? s : 0u; }
  __device__ __forceinline__ uint2 get(uint32_t off) const {
    if constexpr (TLOC == kConst) {
      const CNode n = *reinterpret_cast<const CNode*>(reinterpret_cast<const char*>(c->n) + off);
      return make_uint2(__float_as_uint(n.thr), n.meta);
    } else if constexpr (TLOC == kGlobal) {
      return __ldg(reinterpret_cast<const uint2*>(g + off));
    } else {  // kShared, kSharedReg, kSharedT: absolute shared addresses
      return lds_u2(off);
    }
  }
};

struct DataArgs {
  PipeArgs p;
  const CNode* nodes;          // compact nodes (device global)
  const uint4* wide;           // original 16-byte nodes (kWide)
  uint32_t n_nodes;
  uint32_t abits;              // attr field width (bytes) in compact meta
  const uint32_t* leaf_class;  // null: leaf meta carries the class
  uint32_t* labels;
  uint32_t ns;                 // pipeline stages
  uint32_t tree_bytes;         // shared bytes reserved for the node array (kShared)
  uint32_t stage_bytes;        // stride between stages
  uint32_t record_regs;        // host hint: 8-attribute records walk from registers (kSharedReg)
  uint32_t bulk_tree;          // stage the shared tree with one cp.async.bulk (else per-thread loads)
  uint32_t pdl;                // launched as a programmatic dependent (griddepcontrol)
  uint32_t* depths;            // k_data<DEPTH>: per-record traversal depth (edges root -> leaf)
  // k_data<FRAMES>: resident frame-stream kernel (st_frames_*).  p.m records
  // per frame, frame seq in slot seq % ring (records at rows slot *
  // frame_rows of the tensor map, labels at labels + slot * p.m); control
  // words fctl = {published, closed_at, error, pad} then uint64 done[ring]:
  // tiles of the frames in that slot walked so far (monotone).
  uint32_t* fctl;
  uint32_t ring, frame_rows;
  uint64_t idle_ns;            // a warp waiting this long for a frame stops the stream (error word)
};

// Frame-stream control words (k_data<FRAMES>, st_frames.cu); the uint64
// per-slot completion counters start at word kFDone
enum : uint32_t { kFPublished = 0, kFClosed = 1, kFError = 2, kFDone = 4 };

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Shared-memory carve-out shared by the kernels:
//   [tree | windows (1024-aligned)] [warps x ns stages] [warps x ns mbarriers]
__device__ __forceinline__ uint32_t align1024(uint32_t a) { return (a + 1023u) & ~1023u; }

// ---------------------------------------------------------------------------
// K1: data decomposition
// ---------------------------------------------------------------------------
// One predicated level step of the data walk over a swizzled record tile
// whose record sits inside one 128-byte row (A | 32): if the node is internal,
// node = tb + child + 8*(x[attr] > thr).  bx = row base | in-row XOR mask, so
// the feature address is one LOP3 ((4*attr) ^ bx); leaves stay put with no
// branch and no shared-memory traffic.  Ordered compare, no FTZ (tree.hpp:53).
__device__ __forceinline__ void data_step(uint32_t& thr, uint32_t& meta, uint32_t bx, uint32_t amask,
                                          uint32_t abits) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q;\n\t"
      ".reg .u32 fa, ch;\n\t"
      ".reg .f32 v;\n\t"
      "setp.ge.s32 p, %1, 0;\n\t"
      "and.b32 fa, %1, %3;\n\t"
      "xor.b32 fa, fa, %2;\n\t"
      "@p ld.shared.f32 v, [fa];\n\t"
      "setp.gt.and.f32 q, v, %0, p;\n\t"
      "shr.u32 ch, %1, %4;\n\t"
      "@q add.u32 ch, ch, 8;\n\t"
      "@p ld.shared.v2.u32 {%0, %1}, [ch];\n\t"
      "}"
      : "+f"(*reinterpret_cast<float*>(&thr)), "+r"(meta)
      : "r"(bx), "r"(amask), "r"(abits)
      : "memory");
}

// data_step that also counts the edges taken (traversal depth,
// eval_serial.cpp:77-105): one predicated add on the internal-node predicate.
__device__ __forceinline__ void data_step_d(uint32_t& thr, uint32_t& meta, uint32_t bx, uint32_t amask,
                                            uint32_t abits, uint32_t& depth) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q;\n\t"
      ".reg .u32 fa, ch;\n\t"
      ".reg .f32 v;\n\t"
      "setp.ge.s32 p, %1, 0;\n\t"
      "and.b32 fa, %1, %4;\n\t"
      "xor.b32 fa, fa, %3;\n\t"
      "@p ld.shared.f32 v, [fa];\n\t"
      "setp.gt.and.f32 q, v, %0, p;\n\t"
      "shr.u32 ch, %1, %5;\n\t"
      "@q add.u32 ch, ch, 8;\n\t"
      "@p add.u32 %2, %2, 1;\n\t"
      "@p ld.shared.v2.u32 {%0, %1}, [ch];\n\t"
      "}"
      : "+f"(*reinterpret_cast<float*>(&thr)), "+r"(meta), "+r"(depth)
      : "r"(bx), "r"(amask), "r"(abits)
      : "memory");
}

// Level step over an attribute-major (transposed) tile: the staged meta holds
// 4*attr*R in its low abits_t bits, so the feature address is bx + that
// (bx = tile + 4*record slot): conflict-free, every lane in its own bank.
__device__ __forceinline__ void data_step_t(uint32_t& thr, uint32_t& meta, uint32_t bx, uint32_t amask,
                                            uint32_t abits) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q;\n\t"
      ".reg .u32 fa, ch;\n\t"
      ".reg .f32 v;\n\t"
      "setp.ge.s32 p, %1, 0;\n\t"
      "and.b32 fa, %1, %3;\n\t"
      "add.u32 fa, fa, %2;\n\t"
      "@p ld.shared.f32 v, [fa];\n\t"
      "setp.gt.and.f32 q, v, %0, p;\n\t"
      "shr.u32 ch, %1, %4;\n\t"
      "@q add.u32 ch, ch, 8;\n\t"
      "@p ld.shared.v2.u32 {%0, %1}, [ch];\n\t"
      "}"
      : "+f"(*reinterpret_cast<float*>(&thr)), "+r"(meta)
      : "r"(bx), "r"(amask), "r"(abits)
      : "memory");
}

// Level step with the feature already selected from registers: if the node
// is internal, node = tb + child + 8*(v > thr).
__device__ __forceinline__ void data_step_v(uint32_t& thr, uint32_t& meta, float v, uint32_t abits) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q;\n\t"
      ".reg .u32 ch;\n\t"
      "setp.ge.s32 p, %1, 0;\n\t"
      "setp.gt.and.f32 q, %2, %0, p;\n\t"
      "shr.u32 ch, %1, %3;\n\t"
      "@q add.u32 ch, ch, 8;\n\t"
      "@p ld.shared.v2.u32 {%0, %1}, [ch];\n\t"
      "}"
      : "+f"(*reinterpret_cast<float*>(&thr)), "+r"(meta)
      : "f"(v), "r"(abits)
      : "memory");
}

// x[attr] from A registers (A = 8 or 16): a log2(A)-level select tree on the
// attribute bits of the compact meta (4*attr in the low bits; ptxas turns the
// bit tests into one R2P).  Selects move bits: exact.
template <int A>
__device__ __forceinline__ float pick_reg(const float (&f)[A], uint32_t meta) {
  float v[A];
#pragma unroll
  for (int k = 0; k < A; ++k) v[k] = f[k];
#pragma unroll
  for (int w = A / 2, bit = 4; w >= 1; w /= 2, bit <<= 1) {
    const bool b = meta & (uint32_t)bit;
#pragma unroll
    for (int k = 0; k < w; ++k) v[k] = b ? v[2 * k + 1] : v[2 * k];
  }
  return v[0];
}

// DEPTH: also write each record's traversal depth (edges root -> leaf,
// eval_serial.cpp:77-105) to args.depths; the host never pairs it with the
// register / transposed walks (kSharedReg, kSharedT).
// FRAMES: the resident frame-stream kernel (st_frames_*): the tree is staged
// once, then every warp walks its tiles of frame 0, 1, 2, ... as they are
// published, with no launch and no tree staging per frame (DataArgs.fctl).
template <int A, int S, int TLOC, int LOADER, int CAP, bool DEPTH = false, bool FRAMES = false>
__global__ void __launch_bounds__(kMaxThreads)
    k_data(const DataArgs args, const __grid_constant__ CUtensorMap tmap,
           const __grid_constant__ ConstTree<CAP> ctree) {
  static_assert(!DEPTH || (TLOC != kSharedReg && TLOC != kSharedT), "depth output: record-major walks");
  static_assert(!FRAMES || (LOADER == kTma && !DEPTH), "frame stream: TMA-staged records, labels only");
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int R = 32 * S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nw = blockDim.x >> 5;  // warps in this CTA
  const uint32_t sbase = align1024(smem_u32(smem));

  TreeRef<TLOC, CAP> tree{sbase, reinterpret_cast<const char*>(args.nodes), &ctree};
  uint32_t* labels = args.labels;  // FRAMES: the current frame's label slot

  Pipe<A, S, LOADER> pipe;
  const uint32_t tiles0 = sbase + args.tree_bytes;
  pipe.tiles = tiles0 + (uint32_t)warp * args.ns * args.stage_bytes;
  pipe.bars = tiles0 + nw * args.ns * args.stage_bytes + (uint32_t)warp * args.ns * 8u;
  pipe.stride_bytes = args.stage_bytes;
  pipe.ns = args.ns;
  pipe.tmap = &tmap;
  pipe.p = args.p;
  pipe.lane = lane;

  const uint64_t m = args.p.m;
  const uint64_t n_tiles = (m + R - 1) / R;
  const uint64_t step = (uint64_t)gridDim.x * nw;
  const uint64_t first = (uint64_t)blockIdx.x * nw + warp;
  const uint32_t amask = (1u << args.abits) - 1u;
  constexpr bool kSmemTree = (TLOC == kShared || TLOC == kSharedReg || TLOC == kSharedT);
  const uint4* src = reinterpret_cast<const uint4*>(args.nodes);
  const uint32_t n16 = (args.n_nodes * 8u + 15u) / 16u;
  // The tree bulk copy: one DRAM/L2 round trip for the whole array, in flight
  // beside the first record tiles, then an in-place rebase pass over shared
  // memory (a per-thread ld.global -> st.shared loop serialises one round trip
  // per iteration).  Its mbarrier sits after the per-warp stage barriers,
  // inside the 1024 B alignment reserve of the carve-out.
  const uint32_t tbar = tiles0 + (LOADER == kDirect ? 0u : nw * args.ns * (args.stage_bytes + 8u));
  if (kSmemTree && args.bulk_tree && threadIdx.x == 0) {
    mbar_init(tbar, 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(tbar, 16u * n16);
    bulk_load(sbase, src, 16u * n16, tbar);
  }
  // Programmatic dependent launch (args.pdl): everything above reads only the
  // tree (immutable after st_tree_create) -- records and labels are touched
  // after the previous grid in the stream has completed; dependents may be
  // scheduled from here on (they wait for this grid's completion in turn).
  if (args.pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (args.pdl == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  // first record tiles in flight before the tree is rebased (the TMA does not
  // depend on it); a frame stream only initialises the stage barriers
  pipe.start(first, step, FRAMES ? 0 : n_tiles);

  // ---- stage the node array once per CTA --------------------------------
  constexpr uint32_t kLR = 5u;  // kSharedT: attribute stride 32 records (log2)
  // kSharedT: internal meta = (abs child << abits_t) | 4*attr*32
  const uint32_t abits_t = args.abits + (TLOC == kSharedT ? kLR : 0u);
  if constexpr (kSmemTree) {
    const uint32_t rebase = sbase << args.abits;  // child offset -> absolute address
    if (args.bulk_tree) {
      __syncthreads();  // the barrier's init is visible before anyone waits on it
      mbar_wait(tbar, 0);
      for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) {
        uint4 v = lds_u4(sbase + 16u * i);
        if constexpr (TLOC == kSharedT) {
          if (!(v.y & kLeafBit)) v.y = (((v.y >> args.abits) + sbase) << abits_t) | ((v.y & amask) << kLR);
          if (!(v.w & kLeafBit)) v.w = (((v.w >> args.abits) + sbase) << abits_t) | ((v.w & amask) << kLR);
        } else {
          if (!(v.y & kLeafBit)) v.y += rebase;
          if (!(v.w & kLeafBit)) v.w += rebase;
        }
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sbase + 16u * i), "r"(v.x),
                     "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
      }
    } else {
      for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) {
        uint4 v = __ldg(src + i);
        if constexpr (TLOC == kSharedT) {
          if (!(v.y & kLeafBit)) v.y = (((v.y >> args.abits) + sbase) << abits_t) | ((v.y & amask) << kLR);
          if (!(v.w & kLeafBit)) v.w = (((v.w >> args.abits) + sbase) << abits_t) | ((v.w & amask) << kLR);
        } else {
          if (!(v.y & kLeafBit)) v.y += rebase;
          if (!(v.w & kLeafBit)) v.w += rebase;
        }
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sbase + 16u * i), "r"(v.x),
                     "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
      }
    }
    __syncthreads();
  }

  uint64_t i = 0;
  // FRAMES: the warp walks one continuous tile sequence G = first, first +
  // step, ... over all frames (G = frame * n_tiles + tile of the frame), so
  // frame boundaries fall at different times for different warps and the
  // stage refill runs across them.  A tile is issued once its frame is
  // published (lane 0 caches the published count; a tile whose frame is not
  // published yet is issued when the warp reaches it).  Per frame a warp
  // adds its tile count to the slot's completion counter (one release
  // reduction per frame visited).
  uint64_t G = first;
  uint32_t pub_known = 0, deferred = 0, cur = 0xFFFFFFFFu, cnt = 0;
  auto frame_row = [&](uint64_t g, uint32_t f) -> uint32_t {
    return (f % args.ring) * args.frame_rows + (uint32_t)((g - (uint64_t)f * n_tiles) * R * pipe.arity() / 32u);
  };
  // lane 0: issue tile g into stage s if its frame is published
  auto try_issue = [&](uint64_t g, uint32_t s) -> bool {
    const uint32_t f = (uint32_t)(g / n_tiles);
    if (f >= pub_known) {
      uint32_t pub;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(pub) : "l"(args.fctl + kFPublished) : "memory");
      if (pub > pub_known) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // records arrive through the async proxy
        pub_known = pub;
      }
      if (f >= pub_known) return false;
    }
    const uint32_t bar = pipe.bars + 8u * s;
    mbar_arrive_expect_tx(bar, R * pipe.arity() * 4u);
    tma_load_2d(pipe.stage(s), pipe.tmap, 0, (int)frame_row(g, f), bar);
    return true;
  };
  auto flush_count = [&]() {
    if (cnt) {
      __threadfence();
      __syncwarp();
      if (lane == 0)
        asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(reinterpret_cast<uint64_t*>(args.fctl + kFDone) +
                                                                        cur % args.ring),
                     "l"((uint64_t)cnt)
                     : "memory");
      cnt = 0;
    }
  };
  if constexpr (FRAMES) {
    if (lane == 0)
      for (uint32_t s = 0; s < args.ns; ++s)
        if (!try_issue(first + s * step, s)) deferred |= 1u << s;
    __syncwarp();
  }
  // Done with this warp's i-th tile t: refill its stage with the warp's
  // tile ns further on.
  auto release_tile = [&](uint64_t ii, uint64_t tt) {
    if constexpr (!FRAMES) {
      pipe.release(ii, tt, step, n_tiles);
    } else {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      const uint32_t s = (uint32_t)(ii % args.ns);
      if (lane == 0 && !try_issue(G + args.ns * step, s)) deferred |= 1u << s;
    }
  };
  for (uint64_t t = first;; G += step, t = G, ++i) {
    if constexpr (!FRAMES) {
      if (t >= n_tiles) break;
    } else {
      const uint32_t f = (uint32_t)(G / n_tiles);
      t = G - (uint64_t)f * n_tiles;
      if (f != cur) {  // the previous frame's tiles of this warp are walked: count them now
        flush_count();
        cur = f;
        labels = args.labels + (uint64_t)(f % args.ring) * m;
      }
      const uint32_t s = (uint32_t)(i % args.ns);
      uint32_t ok = 1;
      if (lane == 0 && (deferred >> s) & 1u) {
        // wait for the frame (or the close before it / the idle timeout)
        uint64_t t0 = global_ns();
        uint32_t seen = pub_known;
        while (!try_issue(G, s)) {
          if (pub_known != seen) {  // frames are still arriving: not idle
            seen = pub_known;
            t0 = global_ns();
          }
          uint32_t closed;
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(closed) : "l"(args.fctl + kFClosed) : "memory");
          if (closed <= f) {
            ok = 0;
            break;
          }
          if (global_ns() - t0 > args.idle_ns) {
            atomicOr(args.fctl + kFError, 1u);
            ok = 0;
            break;
          }
          __nanosleep(256);
        }
        if (ok) deferred &= ~(1u << s);
      }
      if (!__shfl_sync(0xffffffffu, ok, 0)) break;
      ++cnt;
    }
    const uint64_t r0 = t * (uint64_t)R;
    const uint32_t tile = pipe.acquire(i, t);
    if constexpr (TLOC == kWide) {
      // generic 16-byte node path: the reference loop (eval_serial.cpp:21-29)
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint32_t r = q * 32 + lane;
        if (r0 + r >= m) continue;
        Rec<A, LOADER> rec;
        rec.init(tile, r, args.p.a, args.p.x, r0 + r, args.p.ld, args.p.layout_soa);
        uint4 nd = __ldg(args.wide);
        uint32_t dep = 0;
        while (nd.w == kNoClass) {
          const uint32_t c = nd.z + (uint32_t)(rec.get(nd.x * 4u) > __uint_as_float(nd.y));
          nd = __ldg(args.wide + c);
          ++dep;
        }
        labels[r0 + r] = nd.w;
        if constexpr (DEPTH) args.depths[r0 + r] = dep;
      }
    } else if constexpr (TLOC == kSharedT && LOADER == kTma && (A == 8 || A == 16)) {
      // transpose the warp's tile in place, one 32-record chunk at a time, to
      // attribute-major: chunk q's (a, lane) at 4*(q*32*A + a*32 + lane) --
      // every later feature read by lane l hits bank l
      // whatever the attribute (the record-major tile puts 128/(4A) records in
      // a row and conflicts on random attributes).  Chunk-local, so only A
      // floats are live at a time.
#pragma unroll
      for (int q = 0; q < S; ++q) {
        float f[A];
        const uint32_t b = (uint32_t)(q * 32 + lane) * (4u * A);
#pragma unroll
        for (int c = 0; c < A / 4; ++c) {
          const uint4 v = lds_u4(tile + swz(b + 16u * c));
          f[4 * c + 0] = __uint_as_float(v.x);
          f[4 * c + 1] = __uint_as_float(v.y);
          f[4 * c + 2] = __uint_as_float(v.z);
          f[4 * c + 3] = __uint_as_float(v.w);
        }
        __syncwarp();
#pragma unroll
        for (int a = 0; a < A; ++a) sts_f32(tile + 4u * (uint32_t)(q * 32 * A + a * 32 + lane), f[a]);
      }
      __syncwarp();
      const uint32_t amask_t = (1u << abits_t) - 1u;
      uint32_t thr[S], meta[S], bx[S];
      const uint2 root = tree.get(tree.root());
#pragma unroll
      for (int q = 0; q < S; ++q) {
        bx[q] = tile + 4u * (uint32_t)(q * 32 * A + lane);
        thr[q] = root.x;
        meta[q] = (r0 + q * 32 + lane < m) ? root.y : kLeafBit;
      }
      while (true) {
        bool any = false;
#pragma unroll
        for (int q = 0; q < S; ++q) any |= (int)meta[q] >= 0;
        if (!any) break;
#pragma unroll
        for (int q = 0; q < S; ++q) data_step_t(thr[q], meta[q], bx[q], amask_t, abits_t);
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {  // folded terminal (unscaled 4*attr in its low bits)
        if (meta[q] & kPairBit) {
          const float v = lds_f32(bx[q] + ((meta[q] & 0x3FFu) << kLR));
          const uint32_t c = (v > __uint_as_float(thr[q])) ? (meta[q] >> 20) : (meta[q] >> 10);
          meta[q] = kLeafBit | (c & 0x3FFu);
        }
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint64_t r = r0 + q * 32 + lane;
        if (r < m) {
          const uint32_t c = meta[q] & ~kLeafBit;
          labels[r] = args.leaf_class ? __ldg(args.leaf_class + c) : c;
        }
      }
    } else if constexpr (TLOC == kSharedReg && LOADER == kTma && (A == 8 || A == 16)) {
      // records -> registers (A/4 conflict-free lds.128 each), tile freed at once
      float f[S][A];
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint32_t b = (uint32_t)(q * 32 + lane) * (4u * A);
#pragma unroll
        for (int c = 0; c < A / 4; ++c) {
          const uint4 v = lds_u4(tile + swz(b + 16u * c));
          f[q][4 * c + 0] = __uint_as_float(v.x);
          f[q][4 * c + 1] = __uint_as_float(v.y);
          f[q][4 * c + 2] = __uint_as_float(v.z);
          f[q][4 * c + 3] = __uint_as_float(v.w);
        }
      }
      release_tile(i, t);  // next tile's TMA overlaps this walk
      uint32_t thr[S], meta[S];
      const uint2 root = tree.get(tree.root());
#pragma unroll
      for (int q = 0; q < S; ++q) {
        thr[q] = root.x;
        meta[q] = (r0 + q * 32 + lane < m) ? root.y : kLeafBit;
      }
      while (true) {
        bool any = false;
#pragma unroll
        for (int q = 0; q < S; ++q) any |= (int)meta[q] >= 0;
        if (!any) break;
#pragma unroll
        for (int q = 0; q < S; ++q) data_step_v(thr[q], meta[q], pick_reg<A>(f[q], meta[q]), args.abits);
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {  // folded terminal: last predicate picks the leaf of the pair
        if (meta[q] & kPairBit) {
          const float v = pick_reg<A>(f[q], meta[q]);
          const uint32_t c = (v > __uint_as_float(thr[q])) ? (meta[q] >> 20) : (meta[q] >> 10);
          meta[q] = kLeafBit | (c & 0x3FFu);
        }
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint64_t r = r0 + q * 32 + lane;
        if (r < m) {
          const uint32_t c = meta[q] & ~kLeafBit;
          labels[r] = args.leaf_class ? __ldg(args.leaf_class + c) : c;
        }
      }
      continue;  // stage already released
    } else if constexpr (TLOC == kShared && LOADER == kTma && Rec<A, LOADER>::kRowLocal) {
      // S independent predicated chains per lane (no per-level branches)
      uint32_t thr[S], meta[S], bx[S], dep[S];
      const uint2 root = tree.get(tree.root());
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint32_t r = q * 32 + lane;
        Rec<A, LOADER> rec;
        rec.init(tile, r, args.p.a, args.p.x, 0, 0, 0);
        bx[q] = rec.base | rec.xm;
        thr[q] = root.x;
        meta[q] = (r0 + r < m) ? root.y : kLeafBit;  // idle slot in the tail tile
        dep[q] = 0;
      }
      while (true) {
        bool any = false;
#pragma unroll
        for (int q = 0; q < S; ++q) any |= (int)meta[q] >= 0;
        if (!any) break;
#pragma unroll
        for (int q = 0; q < S; ++q) {
          if constexpr (DEPTH) data_step_d(thr[q], meta[q], bx[q], amask, args.abits, dep[q]);
          else data_step(thr[q], meta[q], bx[q], amask, args.abits);
        }
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {  // folded terminal: last predicate picks the leaf of the pair
        if (meta[q] & kPairBit) {
          const float v = lds_f32((meta[q] & 0x3FFu) ^ bx[q]);
          const uint32_t c = (v > __uint_as_float(thr[q])) ? (meta[q] >> 20) : (meta[q] >> 10);
          meta[q] = kLeafBit | (c & 0x3FFu);
          dep[q] += 1;  // the terminal's edge to the leaf it picks
        }
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint64_t r = r0 + q * 32 + lane;
        if (r < m) {
          const uint32_t c = meta[q] & ~kLeafBit;
          labels[r] = args.leaf_class ? __ldg(args.leaf_class + c) : c;
          if constexpr (DEPTH) args.depths[r] = dep[q];
        }
      }
    } else if constexpr (S == 1) {
      const uint32_t r = lane;
      const bool valid = r0 + r < m;
      Rec<A, LOADER> rec;
      rec.init(tile, r, args.p.a, args.p.x, r0 + (valid ? r : 0), args.p.ld, args.p.layout_soa);
      uint2 nd = tree.get(tree.root());
      uint32_t meta = valid ? nd.y : kLeafBit;
      float thr = __uint_as_float(nd.x);
      uint32_t dep = 0;
      // Branch-free successor per level: child + (x > thr), as byte offsets.
      while (!(meta & kLeafBit)) {
        const float v = rec.get(meta & amask);
        nd = tree.get((meta >> args.abits) + (v > thr ? 8u : 0u));
        thr = __uint_as_float(nd.x);
        meta = nd.y;
        ++dep;
      }
      if (valid) {
        const uint32_t c = meta & ~kLeafBit;
        labels[r0 + r] = args.leaf_class ? __ldg(args.leaf_class + c) : c;
        if constexpr (DEPTH) args.depths[r0 + r] = dep;
      }
    } else {
      Rec<A, LOADER> rec[S];
      float thr[S];
      uint32_t meta[S], dep[S];
      const uint2 root = tree.get(tree.root());
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint32_t r = q * 32 + lane;
        rec[q].init(tile, r, args.p.a, args.p.x, r0 + (r0 + r < m ? r : 0), args.p.ld, args.p.layout_soa);
        thr[q] = __uint_as_float(root.x);
        meta[q] = (r0 + r < m) ? root.y : kLeafBit;  // idle slot in the tail tile
        dep[q] = 0;
      }
      // Branch-free successor per level: child + (x > thr), as byte offsets.
      while (true) {
        bool any = false;
#pragma unroll
        for (int q = 0; q < S; ++q) {
          if (!(meta[q] & kLeafBit)) {
            const float v = rec[q].get(meta[q] & amask);
            const uint32_t off = (meta[q] >> args.abits) + (v > thr[q] ? 8u : 0u);
            const uint2 nd = tree.get(off);
            thr[q] = __uint_as_float(nd.x);
            meta[q] = nd.y;
            dep[q] += 1;
            any = true;
          }
        }
        if (!any) break;
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint64_t r = r0 + q * 32 + lane;
        if (r < m) {
          const uint32_t c = meta[q] & ~kLeafBit;
          labels[r] = args.leaf_class ? __ldg(args.leaf_class + c) : c;
          if constexpr (DEPTH) args.depths[r] = dep[q];
        }
      }
    }
    release_tile(i, t);
  }
  if constexpr (FRAMES) flush_count();
}

// ---------------------------------------------------------------------------
// K2: speculative decomposition with shfl pointer-jumping
// ---------------------------------------------------------------------------
struct SpecArgs {
  PipeArgs p;
  const SEntry* win;     // window table (device global), padded by 32 entries
  uint32_t n_entries;    // incl. padding
  uint32_t root_code;    // kExitBit | 0 (root window), or kLeafBit|class for N == 1
  uint32_t G;            // lanes per record group (power of two <= 32)
  uint32_t smax;         // doubling steps that resolve every window (fast path)
  uint32_t k;            // EXACT path: check the root after every k doublings
  const uint32_t* leaf_class;
  uint32_t* labels;
  uint32_t* iters;       // EXACT path: per-record counters
  uint32_t* steps;
  uint32_t ns, win_bytes, stage_bytes;
  uint32_t pm_off;       // k_spec_ring SR == 0: path-mask entries (0 = pointer jumping)
  // k_spec_ring CW (8-byte entries), precomputed on the host so the loop
  // reads them straight from the constant bank: attr4 mask, left / right
  // code shifts, code mask, leaf bit, exit payload mask, window stride (8 G)
  uint32_t cw_amask, cw_lsh, cw_rsh, cw_cmask, cw_leaf, cw_emask, cw_wstride;
  // k_spec_ring SL (self-loop codes): terminal-code mask (code bits above
  // log2 G), first leaf code, a stream's advance to its next record (bytes
  // added to / XOR applied to its swizzled record address)
  uint32_t sl_xmask, sl_leafmin, sl_adv, sl_xor;
  uint32_t sl_wmax;      // SL == 3: window steps every record takes (leaves are sinks)
  uint32_t sl_wcheck;    // SL == 3: from this step on, stop once every stream of the warp sits in a sink
  uint32_t sl_ws, sl_wmul;  // entries per window (lanes >= sl_ws read lane 0's); bytes per code unit
  // ring label rows hold raw terminal codes: class = ((code & lab_mask) >>
  // lab_shift) - lab_sub (then the leaf-class table, if any)
  uint32_t lab_mask, lab_shift, lab_sub;
};

// Window codes: lane index (< 32; a width-G shuffle uses its low log2(G)
// bits as the group lane), kExitBit | byte offset of the next
// window's first entry, or kLeafBit | class.  Every lane of a record group
// evaluates its window node's predicate (speculatively: all of them, not
// just the ones on the path), then ceil(log2 h) __shfl_sync pointer-jumping
// steps contract the successor chains inside the group (a single shfl reads
// every source before any lane writes: the snapshot semantics of
// path_double_step, eval_speculative.cpp:38-51); group lane 0 then holds the
// exit.  EXACT reproduces the reference barrier-separated loop and its
// per-record counters: while the root is unresolved apply k doublings
// (eval_speculative.cpp:170-181).
template <int A, int LOADER, bool WIN_SHARED, bool EXACT, int STEPS>
__global__ void __launch_bounds__(kMaxThreads)
    k_spec(const SpecArgs args, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int R = 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nw = blockDim.x >> 5;  // warps in this CTA
  const uint32_t sbase = align1024(smem_u32(smem));

  if constexpr (WIN_SHARED) {
    const uint4* src = reinterpret_cast<const uint4*>(args.win);
    for (uint32_t i = threadIdx.x; i < args.n_entries; i += blockDim.x) {
      const uint4 v = __ldg(src + i);
      asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sbase + 16u * i), "r"(v.x),
                   "r"(v.y), "r"(v.z), "r"(v.w)
                   : "memory");
    }
    __syncthreads();
  }

  Pipe<A, 1, LOADER> pipe;
  const uint32_t tiles0 = sbase + args.win_bytes;
  pipe.tiles = tiles0 + (uint32_t)warp * args.ns * args.stage_bytes;
  pipe.bars = tiles0 + nw * args.ns * args.stage_bytes + (uint32_t)warp * args.ns * 8u;
  pipe.stride_bytes = args.stage_bytes;
  pipe.ns = args.ns;
  pipe.tmap = &tmap;
  pipe.p = args.p;
  pipe.lane = lane;
  // per-warp label (and counter) buffer: one row of 32 records, written
  // coalesced to HBM once per tile
  const uint32_t lbuf = tiles0 + nw * args.ns * (args.stage_bytes + 8u) +
                        (uint32_t)warp * 3u * 128u;

  const uint32_t G = args.G;
  const uint32_t NG = 32u / G;        // record groups per warp
  const uint32_t g = lane / G;        // my group
  const uint32_t j = lane & (G - 1);  // my lane in the group = window-local node
  // byte address of my entry in window 0 (codes carry window byte offsets)
  const uint32_t jaddr = (WIN_SHARED ? sbase : 0u) + 16u * j;
  const char* wglob = reinterpret_cast<const char*>(args.win) + 16u * j;
  const bool root_leaf = (args.root_code & kLeafBit) != 0;

  const uint64_t m = args.p.m;
  const uint64_t n_tiles = (m + R - 1) / R;
  const uint64_t step = (uint64_t)gridDim.x * nw;
  const uint64_t first = (uint64_t)blockIdx.x * nw + warp;
  pipe.start(first, step, n_tiles);

  uint64_t i = 0;
  for (uint64_t t = first; t < n_tiles; t += step, ++i) {
    const uint64_t r0 = t * (uint64_t)R;
    const uint32_t tile = pipe.acquire(i, t);
    const uint32_t rows = (uint32_t)((m - r0) < (uint64_t)R ? (m - r0) : (uint64_t)R);
    if (root_leaf) {  // N == 1: every record is the root's class, zero reductions
      if (lane < rows) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * lane), "r"(args.root_code) : "memory");
        if constexpr (EXACT) {
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 128u + 4u * lane), "r"(0u) : "memory");
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 256u + 4u * lane), "r"(0u) : "memory");
        }
      }
    } else {
      // Group g classifies tile rows g, g+NG, ...; a finished group refills
      // with its next row immediately, so skewed depths do not idle it.
      uint32_t r = g;
      bool active = r < rows;
      uint32_t woff = 0;  // byte offset of the current window
      uint32_t n_it = 0, n_st = 0;
      Rec<A, LOADER> rec;
      rec.init(tile, active ? r : 0u, args.p.a, args.p.x, r0 + (active ? r : 0u), args.p.ld, args.p.layout_soa);
      do {
        // -- node evaluation: every window lane computes its successor ------
        uint4 e;
        if constexpr (WIN_SHARED) e = lds_u4(jaddr + woff);
        else e = __ldg(reinterpret_cast<const uint4*>(wglob + woff));
        const float v = rec.get(e.y & 0x00FFFFFFu);
        uint32_t c = (v > __uint_as_float(e.x)) ? e.w : e.z;
        // -- path reduction: shfl pointer-jumping inside the group ----------
        if constexpr (!EXACT) {
          if constexpr (STEPS >= 0) {
#pragma unroll
            for (int s = 0; s < STEPS; ++s) {
              const uint32_t u = __shfl_sync(0xffffffffu, c, c, G);
              c = (c < 32u) ? u : c;
            }
          } else {
            for (uint32_t s = 0; s < args.smax; ++s) {
              const uint32_t u = __shfl_sync(0xffffffffu, c, c, G);
              c = (c < 32u) ? u : c;
            }
          }
        } else {
          // Every group (idle ones included) doubles until its root is
          // resolved, so its exit code is a valid window offset; only active
          // groups count.
          while (true) {
            const uint32_t rt = __shfl_sync(0xffffffffu, c, 0, G);
            const bool need = rt < 32u;
            if (!__any_sync(0xffffffffu, need)) break;
            for (uint32_t s = 0; s < args.k; ++s) {
              const uint32_t u = __shfl_sync(0xffffffffu, c, c, G);
              if (need && c < 32u) c = u;
            }
            if (need && active) {
              n_it += 1;
              n_st += args.k;
            }
          }
        }
        const uint32_t root = __shfl_sync(0xffffffffu, c, 0, G);
        if (root & kLeafBit) {
          if (active && j == 0) {
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * r), "r"(root) : "memory");
            if constexpr (EXACT) {
              asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 128u + 4u * r), "r"(n_it) : "memory");
              asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 256u + 4u * r), "r"(n_st) : "memory");
            }
          }
          n_it = n_st = 0;
          r += NG;
          active = r < rows;
          woff = 0;
          // idle groups keep walking their last record (finite, never stored)
          if (active) rec.advance(r, NG, args.p.a, tile, args.p.x, r0 + r, args.p.ld, args.p.layout_soa);
        } else {
          woff = root & ~kExitBit;
        }
      } while (__any_sync(0xffffffffu, active));
    }
    __syncwarp();
    if (lane < rows) {
      uint32_t code;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(code) : "r"(lbuf + 4u * lane));
      const uint32_t cls = code & ~kLeafBit;
      args.labels[r0 + lane] = args.leaf_class ? __ldg(args.leaf_class + cls) : cls;
      if constexpr (EXACT) {
        uint32_t a, b;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a) : "r"(lbuf + 128u + 4u * lane));
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(b) : "r"(lbuf + 256u + 4u * lane));
        args.iters[r0 + lane] = a;
        args.steps[r0 + lane] = b;
      }
    }
    pipe.release(i, t, step, n_tiles);
  }
}

// ---------------------------------------------------------------------------
// K2r: speculative decomposition over a CTA-shared tile ring
// ---------------------------------------------------------------------------
// Same per-window algorithm as k_spec (fast fixed-step path), but the record
// staging is decoupled from the warp count: the CTA owns a ring of NS tile
// slots; warps take tiles in ticket order (shared-memory counter) and the warp
// that finishes tile k refills the same slot with tile k + NS (TMA, or a
// warp-cooperative store for the one partial tail tile) -- no producer to
// block behind a slow tile.  The speculative walk is latency-bound, so this
// buys ~1.7x the resident warps for the same shared memory (only the tiles
// DRAM latency needs are in flight, not two per warp).
struct SpecRingArgs {
  SpecArgs s;
  uint32_t n_slots;       // NS
  uint32_t ns_magic;      // floor(2^32 / NS): ticket -> (generation, slot) without a division
  uint32_t bulk_win;      // stage the window table with one cp.async.bulk (else per-thread loads)
  // FR (frame stream, st_frames_* with the speculative algorithm): s.p.m
  // records per frame in tpf tiles, frame f in slot f % ring (tensor-map rows
  // from slot * frame_rows, labels from s.labels + slot * s.p.m), control
  // words as DataArgs.fctl
  uint32_t* fctl;
  uint32_t ring, frame_rows;
  uint64_t tpf, idle_ns;
  uint32_t tile_mult;     // host: records per ring slot / 32 (the kernel's RT); 0 = lane triples
  uint32_t triple;        // host: lane-triple slots of kTripleSlot (1) or 3/2 kTripleSlot (3) records
};

// RT: records per ring slot / 32.  Two-stream groups over 64-record slots
// (RT = 2) walk 4 records per stream instead of 2, which evens out the
// streams' window counts on skewed trees and halves the per-slot overhead.
// SL: self-loop terminal codes (WinTable::sl_*): a pointer-jumping step is
// one shfl with no select.  With SR == 2: SL == 1 advances a resolved
// stream by a constant address step under predication (skewed trees, where
// some stream of the warp resolves in almost every window step), SL == 2 in
// a divergent branch taken only when one does; SL == 3 runs every record for
// a fixed sl_wmax window steps with leaves as absorbing sink windows -- no
// per-step test at all (balanced trees, where records' window counts barely
// differ).
// L3: interleaved lane triples (fixed-trip loop, G = 4 self-loop tables of
// three-node windows): lanes 3g .. 3g + 2 hold window lanes 0..2 of record
// group g < 10, so a warp instruction carries 10 records instead of 8 (the
// fourth lane of a 4-lane group only ever mirrors lane 0); a doubling step's
// source lane is 3g + (code & 3).  Lanes 30 / 31 mirror lanes 27 / 28 (same
// addresses: broadcasts, no extra wavefronts).  80-record ring slots (8 per
// group).
// FR: the resident frame stream.  The CTA's tickets continue across frames
// (tile G = blockIdx + ticket * grid of the endless frame sequence); a warp
// waits for a ticket's frame to be published before touching its slot, and
// a slot whose next tile lies in a frame not yet published is handed over
// "deferred" (generation word bit 0): the warp that takes that ticket issues
// its TMA itself.  Per frame visited a warp adds its walked-tile count to the
// slot's completion counter (as k_data<FRAMES>).
template <int A, bool WIN_SHARED, int STEPS, int SR, bool CW = false, int RT = 1, int SL = 0, int L3 = 0,
          bool FR = false>
__global__ void __launch_bounds__(kMaxThreads)
    k_spec_ring(const SpecRingArgs ra, const __grid_constant__ CUtensorMap tmap) {
  static_assert(!FR || (SL == 3 && RT == 1), "frame stream: fixed-trip loop, one-chunk slots");
  static_assert(!CW || (WIN_SHARED && SR >= 1), "8-byte windows: shared table, window-loop paths");
  static_assert(!SL || SR == 0 || (SR == 2 && CW), "self-loop codes: one window, or two 8-byte-window streams");
  static_assert(SL < 2 || SR == 2, "branchy / fixed-trip stream loops: two-stream layout");
  static_assert(RT == 1 || SR == 2, "multi-chunk slots: two-stream loop only");
  static_assert(!L3 || (SL == 3 && RT == 1), "lane triples: fixed-trip loop, 80-record slots");
  extern __shared__ __align__(1024) unsigned char smem[];
  const SpecArgs& args = ra.s;
  constexpr int R = L3 ? (L3 == 3 ? kTripleSlot * 3 / 2 : kTripleSlot) : 32 * RT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t NS = ra.n_slots;
  const uint32_t sbase = align1024(smem_u32(smem));

  // [windows] [NS slots] [full bars] [slot generations] [ticket] [per-warp label rows]
  const uint32_t slots0 = sbase + args.win_bytes;
  const uint32_t full0 = slots0 + NS * args.stage_bytes;
  const uint32_t gen0 = full0 + 8u * NS;
  const uint32_t ticket = gen0 + ((4u * NS + 15u) & ~15u);
  uint32_t lbuf;  // opaque copy: keeps the per-warp label row in a register (no S2R remat in the walk)
  asm("mov.u32 %0, %1;" : "=r"(lbuf) : "r"(ticket + 16u + (uint32_t)warp * (4u * R)));

  const uint64_t m = args.p.m;
  const uint64_t n_tiles = (m + R - 1) / R;
  const uint64_t my_tiles = blockIdx.x < n_tiles ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint32_t a_rt = A > 0 ? (uint32_t)A : args.p.a;
  auto tile_of = [&](uint64_t j) { return blockIdx.x + j * (uint64_t)gridDim.x; };
  // Stage tile j into slot b: TMA for full tiles (lane 0), warp-cooperative
  // swizzled stores + a plain arrive for the partial tail.
  // ticket -> (generation q, slot r): multiply-high estimate, one correction
  auto divmod_ns = [&](uint32_t x, uint32_t& q, uint32_t& r) {
    q = __umulhi(x, ra.ns_magic);
    r = x - q * NS;
    if (r >= NS) ++q, r -= NS;
  };
  auto fill = [&](uint64_t jj, uint32_t b) {
    const uint64_t t = tile_of(jj);
    const uint32_t dst = slots0 + b * args.stage_bytes;
    const uint64_t r0 = t * (uint64_t)R;
    if ((t + 1) * (uint64_t)R <= m) {
      if (lane == 0) {
        mbar_arrive_expect_tx(full0 + 8u * b, R * a_rt * 4u);
        tma_load_2d(dst, &tmap, 0, (int)(r0 * a_rt / 32u), full0 + 8u * b);
      }
    } else {
      const uint32_t rows = (uint32_t)(m - r0);
      for (uint32_t f = lane; f < rows * a_rt; f += 32) {
        const uint32_t r = f / a_rt, aa = f - r * a_rt;
        sts_f32(dst + swz(f * 4u), __ldg(args.p.x + (r0 + r) * (uint64_t)args.p.ld + aa));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(full0 + 8u * b);
    }
  };

  // FR: frame of a tile, its tensor-map row, publication (lane 0 caches it)
  uint32_t pub_known = 0, cur = 0xFFFFFFFFu, cnt = 0;
  auto fr_published = [&](uint32_t f) -> bool {  // lane 0
    if (f < pub_known) return true;
    uint32_t pub;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(pub) : "l"(ra.fctl + kFPublished) : "memory");
    if (pub > pub_known) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      pub_known = pub;
    }
    return f < pub_known;
  };
  auto fr_issue = [&](uint64_t jj, uint32_t b) {  // lane 0, frame published
    const uint64_t G = tile_of(jj);
    const uint32_t f = (uint32_t)(G / ra.tpf);
    const uint32_t row = (f % ra.ring) * ra.frame_rows + (uint32_t)((G - (uint64_t)f * ra.tpf) * R * a_rt / 32u);
    mbar_arrive_expect_tx(full0 + 8u * b, R * a_rt * 4u);
    tma_load_2d(slots0 + b * args.stage_bytes, &tmap, 0, (int)row, full0 + 8u * b);
  };
  auto fr_try_fill = [&](uint64_t jj, uint32_t b) -> bool {  // lane 0
    if (!fr_published((uint32_t)(tile_of(jj) / ra.tpf))) return false;
    fr_issue(jj, b);
    return true;
  };
  auto flush_count = [&]() {
    if (cnt) {
      __threadfence();
      __syncwarp();
      if (lane == 0)
        asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(reinterpret_cast<uint64_t*>(ra.fctl + kFDone) +
                                                                        cur % ra.ring),
                     "l"((uint64_t)cnt)
                     : "memory");
      cnt = 0;
    }
  };

  if (threadIdx.x == 0) {
    for (uint32_t b = 0; b < NS; ++b) {
      mbar_init(full0 + 8u * b, 1);
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(gen0 + 4u * b), "r"(0u) : "memory");
    }
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(ticket), "r"(0u) : "memory");
    if (WIN_SHARED && ra.bulk_win) mbar_init(ticket + 8u, 1);
    fence_barrier_init();
    if (WIN_SHARED && ra.bulk_win) {  // the whole table in one round trip
      mbar_arrive_expect_tx(ticket + 8u, 16u * args.n_entries);
      bulk_load(sbase, args.win, 16u * args.n_entries, ticket + 8u);
    }
  }
  __syncthreads();
  if constexpr (FR) {
    // generation words: gen << 1 | deferred (the taker of that ticket issues the TMA)
    if (warp == 0 && lane == 0)
      for (uint32_t b = 0; b < NS; ++b)
        if (!fr_try_fill(b, b)) asm volatile("st.shared.u32 [%0], %1;" ::"r"(gen0 + 4u * b), "r"(1u) : "memory");
  } else if (warp == 0) {
    for (uint64_t jj = 0; jj < NS && jj < my_tiles; ++jj) fill(jj, (uint32_t)jj);
  }
  // window table staged while the first tiles are in flight
  if constexpr (WIN_SHARED) {
    if (!ra.bulk_win) {
      const uint4* src = reinterpret_cast<const uint4*>(args.win);
      for (uint32_t i = threadIdx.x; i < args.n_entries; i += blockDim.x) {
        const uint4 v = __ldg(src + i);
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sbase + 16u * i), "r"(v.x),
                     "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
      }
    }
  }

  const uint32_t G = args.G;
  const uint32_t NG = L3 ? 10u : 32u / G;
  const uint32_t g = L3 ? (lane < 30 ? (uint32_t)lane / 3u : 9u) : lane / G;
  const uint32_t j = L3 ? (lane < 30 ? (uint32_t)lane - 3u * g : (uint32_t)lane - 30u) : lane & (G - 1);
  // self-loop tables pack sl_ws entries per window (G = 4: the 3 nodes of a
  // two-level window, 24 B); lanes beyond them read lane 0's entry (a
  // broadcast, never on a path)
  const uint32_t jaddr =
      (WIN_SHARED ? sbase : 0u) + (CW ? 8u : 16u) * ((CW && SL >= 1) ? (j < args.sl_ws ? j : 0u) : j);
  const char* wglob = reinterpret_cast<const char*>(args.win) + 16u * j;
  if constexpr (WIN_SHARED) {  // window table staged
    if (ra.bulk_win) mbar_wait(ticket + 8u, 0);
    // a CTA barrier either way: after the per-thread spin alone the compiler
    // can no longer prove the warp converged and moves the loop's warp-uniform
    // values off the uniform datapath (+20 % SASS in the window loop)
    __syncthreads();
  }
  // Window entry formats.  16-byte SEntry, or (CW) 8-byte {thr, attr4 |
  // left << cw_abits | right << (cw_abits + cw_cbits)} with cw_cbits-bit
  // codes: lane (< 32), exit (bit cbits-2 | window index; windows are G
  // entries apart), leaf (bit cbits-1 | class): half the shared-memory
  // wavefronts of the entry loads.
  struct Ent { uint32_t thr, w, l, r; };
  const uint32_t leafbit = CW ? args.cw_leaf : kLeafBit;
  // CW: `woff` is the window index (entry address = one IMAD); otherwise a
  // byte offset
  auto load_ent = [&](uint32_t woff) -> Ent {
    if constexpr (CW) {
      const uint2 t = lds_u2(jaddr + woff * args.cw_wstride);
      return {t.x, t.y, 0u, 0u};
    } else {
      uint4 t;
      if constexpr (WIN_SHARED) t = lds_u4(jaddr + woff);
      else t = __ldg(reinterpret_cast<const uint4*>(wglob + woff));
      return {t.x, t.y, t.z, t.w};
    }
  };
  auto ent_attr4 = [&](const Ent& e) -> uint32_t {
    if constexpr (CW) return e.w & args.cw_amask;
    else return e.w & 0x00FFFFFFu;
  };
  auto ent_next = [&](const Ent& e, bool right) -> uint32_t {
    if constexpr (CW) return right ? (e.w >> args.cw_rsh) : ((e.w >> args.cw_lsh) & args.cw_cmask);
    else return right ? e.r : e.l;
  };
  auto exit_off = [&](uint32_t root) -> uint32_t {
    if constexpr (CW) return root & args.cw_emask;
    else return root & ~kExitBit;
  };
  // SR == 0: the whole tree is one window (the paper's Proc. 5 geometry):
  // each lane's entry is the same for every record -- load it once.
  uint4 e1 = make_uint4(0u, 0u, 0u, 0u), pm1 = make_uint4(0u, 0u, 0u, 0u);
  if constexpr (SR == 0) {
    static_assert(SR != 0 || WIN_SHARED, "one-window path stages its table in shared memory");
    // SL: the self-loop copy of the window (host offset in pm_off)
    e1 = SL ? lds_u4(sbase + 16u * (args.pm_off + j)) : lds_u4(jaddr);
    if (args.pm_off && !SL) pm1 = lds_u4(sbase + 16u * (args.pm_off + j));
  }

  while (true) {
    uint32_t tk = 0;
    if (lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(tk) : "r"(ticket) : "memory");
    tk = __shfl_sync(0xffffffffu, tk, 0);
    uint64_t t;
    uint32_t* labels = args.labels;
    if constexpr (FR) {
      const uint64_t Gt = tile_of(tk);
      const uint32_t f = (uint32_t)(Gt / ra.tpf);
      t = Gt - (uint64_t)f * ra.tpf;
      if (f != cur) {  // this warp's tiles of the previous frame are walked: count them
        flush_count();
        cur = f;
      }
      labels = args.labels + (uint64_t)(f % ra.ring) * m;
      // the ticket's frame must be out (or the stream closed before it / idle)
      uint32_t ok = 1;
      if (lane == 0 && !fr_published(f)) {
        uint64_t t0 = global_ns();
        uint32_t seen = pub_known;
        while (!fr_published(f)) {
          if (pub_known != seen) {
            seen = pub_known;
            t0 = global_ns();
          }
          uint32_t closed;
          asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(closed) : "l"(ra.fctl + kFClosed) : "memory");
          if (closed <= f) {
            ok = 0;
            break;
          }
          if (global_ns() - t0 > ra.idle_ns) {
            atomicOr(ra.fctl + kFError, 1u);
            ok = 0;
            break;
          }
          __nanosleep(256);
        }
      }
      if (!__shfl_sync(0xffffffffu, ok, 0)) break;
      ++cnt;
    } else {
      if (tk >= my_tiles) break;
      t = tile_of(tk);
    }
    const uint64_t r0 = t * (uint64_t)R;
    uint32_t gen, b;
    divmod_ns(tk, gen, b);
    const uint32_t tile = slots0 + b * args.stage_bytes;
    const uint32_t rows = (uint32_t)((m - r0) < (uint64_t)R ? (m - r0) : (uint64_t)R);
    // A parity wait cannot tell generation g of a slot from g + 2: a slow
    // warp may still hold ticket tk - NS (slot b not yet refilled for tk)
    // while faster warps have taken every ticket up to tk.  So first wait
    // until the refill for generation tk / NS has been issued (the warp that
    // finished tk - NS publishes it), then the parity wait is unambiguous.
    // The generation word only gates *which* phase to wait for; the tile's
    // bytes are published by the mbarrier (complete_tx, acquire on the wait),
    // so plain volatile shared accesses suffice.
    // Every lane polls the same word (one broadcast wavefront, warp-uniform
    // exit): no divergent lane-0 section before the walk's shuffles.
    if constexpr (FR) {
      uint32_t have;
      do {
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(have) : "r"(gen0 + 4u * b) : "memory");
      } while (__any_sync(0xffffffffu, (have >> 1) < gen));
      // handed over deferred: the frame was not out when the slot was freed
      if (have == ((gen << 1) | 1u) && lane == 0) fr_issue(tk, b);
      __syncwarp();
    } else {
      uint32_t have;
      do {
        asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(have) : "r"(gen0 + 4u * b) : "memory");
      } while (__any_sync(0xffffffffu, have < gen));
    }
    mbar_wait(full0 + 8u * b, gen & 1u);
    if (args.root_code & kLeafBit) {  // N == 1
#pragma unroll
      for (int k = 0; k < (R + 31) / 32; ++k)
        if (lane + 32u * k < rows)
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * (lane + 32u * k)), "r"(args.root_code)
                       : "memory");
    } else if constexpr (SR == 0) {
      // One window: every record resolves in one pass, so the passes over
      // the tile's records are independent chains (feature load -> compare
      // -> doubling shuffles -> root) the compiler interleaves.  Rows past a
      // partial tile's end re-read the last row and are never stored.
      const uint32_t thr = e1.x, attr4 = e1.y & 0x00FFFFFFu;
      auto feature = [&](uint32_t r) {
        const uint32_t rr = r < rows ? r : rows - 1u;
        if constexpr (Rec<A, kTma>::kRowLocal) {
          const uint32_t ra4 = rr * (4u * (uint32_t)A), rowb = ra4 & ~127u;
          return lds_f32(attr4 ^ ((tile + rowb) | (((rowb >> 3) & 0x70u) ^ (ra4 & 127u))));
        } else {
          Rec<A, kTma> rec;
          rec.init(tile, rr, args.p.a, args.p.x, 0, 0, 0);
          return rec.get(attr4);
        }
      };
      if constexpr (SL) {
        // Pointer jumping with self-loop leaf codes: a leaf code's low bits
        // name its own lane, so each doubling is one shfl with no select
        // (snapshot semantics of path_double_step, eval_speculative.cpp:
        // 38-51); group lane 0 then holds the leaf.  Full tiles advance the
        // feature / label addresses by constants (no row clamp).
        if (rows == 32u * RT) {
          const uint32_t a4 = 4u * (A > 0 ? (uint32_t)A : args.p.a);
          const uint32_t df = NG * a4, dl = 4u * NG;
          uint32_t f = tile + g * a4 + attr4, la = lbuf + 4u * g;
#pragma unroll 4
          for (uint32_t r = g; r < 32u * RT; r += NG, f += df, la += dl) {
            const float v = lds_f32(f ^ ((f >> 3) & 0x70u));  // swizzled (tile 1024-aligned)
            uint32_t c = (v > __uint_as_float(thr)) ? e1.w : e1.z;
#pragma unroll
            for (int st = 0; st < (STEPS > 0 ? STEPS : 0); ++st) c = __shfl_sync(0xffffffffu, c, c, G);
            // group lane 0 holds the root's contracted code: no broadcast
            if (j == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(la), "r"(c) : "memory");
          }
        } else {
#pragma unroll 4
          for (uint32_t r = g; r < 32u * RT; r += NG) {
            const float v = feature(r);
            uint32_t c = (v > __uint_as_float(thr)) ? e1.w : e1.z;
#pragma unroll
            for (int st = 0; st < (STEPS > 0 ? STEPS : 0); ++st) c = __shfl_sync(0xffffffffu, c, c, G);
            if (j == 0 && r < rows)
              asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * r), "r"(c) : "memory");
          }
        }
      } else if (args.pm_off) {
        // Ballot reduction: one vote gathers every lane's predicate (the
        // same speculation), and the lane whose leaf path mask matches --
        // exactly one per group in a tree -- stores its class.  No shuffles.
        const uint32_t gsh = g * G;
        if (rows == 32u) {
          // full tile (warp-uniform): no row clamp, the feature and label
          // addresses advance by a constant per record, and the path masks
          // are pre-shifted to the group's lanes -- the loop is issue-bound,
          // so every instruction per record counts
          const uint32_t want = pm1.w << gsh, care = pm1.z << gsh;
          const bool has_leaf = pm1.y != 0u;
          const uint32_t a4 = 4u * (A > 0 ? (uint32_t)A : args.p.a);
          const uint32_t df = NG * a4, dl = 4u * NG;
          uint32_t f = tile + g * a4 + attr4, la = lbuf + 4u * g;
#pragma unroll 4
          for (uint32_t r = g; r < 32u; r += NG, f += df, la += dl) {
            const float v = lds_f32(f ^ ((f >> 3) & 0x70u));  // swizzled (tile 1024-aligned)
            const uint32_t preds = __ballot_sync(0xffffffffu, v > __uint_as_float(thr));
            if (has_leaf && ((preds ^ want) & care) == 0u)
              asm volatile("st.shared.u32 [%0], %1;" ::"r"(la), "r"(pm1.y) : "memory");
          }
        } else {
#pragma unroll 4
          for (uint32_t r = g; r < 32u; r += NG) {
            const float v = feature(r);
            const uint32_t preds = __ballot_sync(0xffffffffu, v > __uint_as_float(thr)) >> gsh;
            if (pm1.y != 0u && ((preds ^ pm1.w) & pm1.z) == 0u && r < rows)
              asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * r), "r"(pm1.y) : "memory");
          }
        }
      } else {
#pragma unroll 4
        for (uint32_t r = g; r < 32u; r += NG) {
          const float v = feature(r);
          uint32_t c = (v > __uint_as_float(thr)) ? e1.w : e1.z;
          if constexpr (STEPS >= 0) {
#pragma unroll
            for (int st = 0; st < STEPS; ++st) {
              const uint32_t u = __shfl_sync(0xffffffffu, c, c, G);
              c = (c < 32u) ? u : c;
            }
          } else {
            for (uint32_t st = 0; st < args.smax; ++st) {
              const uint32_t u = __shfl_sync(0xffffffffu, c, c, G);
              c = (c < 32u) ? u : c;
            }
          }
          if (j == 0 && r < rows)  // group lane 0 holds the root's code
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * r), "r"(c) : "memory");
        }
      }
    } else if constexpr (SR == 1) {
      // One record stream per group: the lean loop.  A group whose rows are
      // exhausted keeps re-walking its last record (finite, never stored):
      // its extra loads cost less than predicating every step.
      constexpr bool kRowLocal = Rec<A, kTma>::kRowLocal;
      const uint32_t a4 = 4u * (A > 0 ? (uint32_t)A : args.p.a);
      uint32_t r = g;
      bool active = r < rows;
      uint32_t woff = 0, bx = 0;
      Rec<A, kTma> rec;
      if constexpr (kRowLocal) {
        const uint32_t ra4 = (active ? r : 0u) * a4, rowb = ra4 & ~127u;
        bx = (tile + rowb) | (((rowb >> 3) & 0x70u) ^ (ra4 & 127u));
      } else {
        rec.init(tile, active ? r : 0u, args.p.a, args.p.x, 0, 0, 0);
      }
      do {
        const Ent e = load_ent(woff);
        float v;
        if constexpr (kRowLocal) v = lds_f32(ent_attr4(e) ^ bx);
        else v = rec.get(ent_attr4(e));
        uint32_t c = ent_next(e, v > __uint_as_float(e.thr));
        if constexpr (STEPS >= 0) {
#pragma unroll
          for (int st = 0; st < STEPS; ++st) {
            const uint32_t u = __shfl_sync(0xffffffffu, c, c, G);
            c = (c < 32u) ? u : c;
          }
        } else {
          for (uint32_t st = 0; st < args.smax; ++st) {
            const uint32_t u = __shfl_sync(0xffffffffu, c, c, G);
            c = (c < 32u) ? u : c;
          }
        }
        const uint32_t root = __shfl_sync(0xffffffffu, c, 0, G);
        if (root & leafbit) {
          if (active && j == 0)
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * r), "r"(root) : "memory");
          r += NG;
          active = r < rows;
          woff = 0;
          if (active) {
            if constexpr (kRowLocal) {
              const uint32_t ra4 = r * a4, rowb = ra4 & ~127u;
              bx = (tile + rowb) | (((rowb >> 3) & 0x70u) ^ (ra4 & 127u));
            } else {
              rec.init(tile, r, args.p.a, args.p.x, 0, 0, 0);
            }
          }
        } else {
          woff = exit_off(root);
        }
      } while (__any_sync(0xffffffffu, active));
    } else if constexpr (SR == 2 && SL == 3) {
      // Fixed trip count (the paper's Proc. 5 property lifted to windows:
      // terminal codes are fixpoints, so extra steps are harmless): each
      // group walks its records as batches of KS independent streams, every
      // stream exactly sl_wmax window steps -- entry, feature, compare,
      // shift, select-free doublings, root broadcast, mask, LEA -- then the
      // group's lane 0 stores the KS leaf codes.  No leaf test, no stream
      // state, no divergence.
      static_assert(Rec<A, kTma>::kRowLocal, "fixed-trip streams: records inside one 128-byte row");
      // 4 streams per batch (8 per triple measured even on C5, +4 % on C3)
      constexpr int KS = 4;
      const uint32_t NL = L3 ? 3u : G;  // lanes per group: lane s % NL stores stream s
      const uint32_t a4 = 4u * (uint32_t)A;
      auto base_of = [&](uint32_t rr) {
        const uint32_t ra4 = rr * a4, rowb = ra4 & ~127u;
        return (tile + rowb) | (((rowb >> 3) & 0x70u) ^ (ra4 & 127u));
      };
      const uint32_t per_group = R / NG;  // records of this group in the slot
      const uint32_t g3 = 3u * g;         // L3: the group's lane 0
      // every stream starts in the root window: its entry lives in registers
      const uint2 e_root = lds_u2(jaddr);
      for (uint32_t k0 = 0; k0 < per_group; k0 += KS) {
        uint32_t rr[KS], bx[KS], ad[KS], c[KS];
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          rr[s] = g + NG * (k0 + s);
          bx[s] = base_of(rr[s] < rows ? rr[s] : 0u);  // rows past a partial tile walk record 0
        }
        auto step = [&](const bool first) {
#pragma unroll
          for (int s = 0; s < KS; ++s) {
            const uint2 e = first ? e_root : lds_u2(ad[s]);
            const float v = lds_f32((e.y & args.cw_amask) ^ bx[s]);
            c[s] = e.y >> (v > __uint_as_float(e.x) ? args.cw_rsh : args.cw_lsh);
          }
          // one pointer-jumping step: width-G segments, or (L3) source lane
          // 3g + the code's lane bits
          auto jump = [&](uint32_t cc) -> uint32_t {
            if constexpr (L3) return __shfl_sync(0xffffffffu, cc, g3 + (cc & 3u));
            else return __shfl_sync(0xffffffffu, cc, cc, G);
          };
          if constexpr (STEPS >= 0) {
#pragma unroll
            for (int st = 0; st < STEPS; ++st)
#pragma unroll
              for (int s = 0; s < KS; ++s) c[s] = jump(c[s]);
          } else {
            for (uint32_t st = 0; st < args.smax; ++st)
#pragma unroll
              for (int s = 0; s < KS; ++s) c[s] = jump(c[s]);
          }
#pragma unroll
          for (int s = 0; s < KS; s += 2) {  // one root broadcast per two streams
            const uint32_t v = L3 ? __shfl_sync(0xffffffffu, pack_lo16(c[s], c[s + 1]), g3)
                                  : __shfl_sync(0xffffffffu, pack_lo16(c[s], c[s + 1]), 0, G);
            const uint32_t x0 = v & args.sl_xmask, x1 = (v >> 16) & args.sl_xmask;
            ad[s] = jaddr + x0 * args.sl_wmul;
            ad[s + 1] = jaddr + x1 * args.sl_wmul;
            c[s] = x0;
            c[s + 1] = x1;
          }
        };
        step(true);
        for (uint32_t w = 1; w < args.sl_wmax; ++w) {
          // skewed trees: the warp's batch ends when all its streams are
          // absorbed (one vote per step, from step sl_wcheck on) instead of
          // after the deepest record's window count
          if (w >= args.sl_wcheck) {
            bool sunk = true;
#pragma unroll
            for (int s = 0; s < KS; ++s) sunk &= c[s] >= args.sl_leafmin;
            if (__all_sync(0xffffffffu, sunk)) break;
          }
          step(false);
        }
        // lane s % NL of the group stores stream s (every stream stored even
        // when the group has fewer lanes than streams: G = 2); mirror lanes none
        const bool st_ok = L3 ? lane < 30 : true;
#pragma unroll
        for (int s = 0; s < KS; ++s)
          if (st_ok && j == (uint32_t)s % NL && rr[s] < rows)
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * rr[s]), "r"(c[s]) : "memory");
      }
    } else if constexpr (SR == 2 && SL == 2) {
      // Two record streams, self-loop codes, the stream advance in a
      // divergent branch (taken by the warp only in steps where some stream
      // resolves).
      static_assert(Rec<A, kTma>::kRowLocal, "self-loop streams: records inside one 128-byte row");
      const uint32_t a4 = 4u * (uint32_t)A;
      auto base_of = [&](uint32_t rr) {
        const uint32_t ra4 = rr * a4, rowb = ra4 & ~127u;
        return (tile + rowb) | (((rowb >> 3) & 0x70u) ^ (ra4 & 127u));
      };
      uint32_t rA = g, rB = g + NG;
      bool aA = rA < rows, aB = rB < rows;
      uint32_t wA = 0, wB = 0;
      uint32_t bA = base_of(aA ? rA : 0u), bB = base_of(aB ? rB : 0u);
      // lane j of the group collects the code of its stream's j-th record in
      // a register (no shared-memory store per resolution); stored at the end
      const uint32_t mA = g + 2u * NG * j, mB = mA + NG;
      uint32_t kA = 0u, kB = 0u;
      do {
        const uint2 eA = lds_u2(jaddr + wA), eB = lds_u2(jaddr + wB);
        const float vA = lds_f32((eA.y & args.cw_amask) ^ bA), vB = lds_f32((eB.y & args.cw_amask) ^ bB);
        uint32_t cA = eA.y >> (vA > __uint_as_float(eA.x) ? args.cw_rsh : args.cw_lsh);
        uint32_t cB = eB.y >> (vB > __uint_as_float(eB.x) ? args.cw_rsh : args.cw_lsh);
        if constexpr (STEPS >= 0) {
#pragma unroll
          for (int st = 0; st < STEPS; ++st) {
            cA = __shfl_sync(0xffffffffu, cA, cA, G);
            cB = __shfl_sync(0xffffffffu, cB, cB, G);
          }
        } else {
          for (uint32_t st = 0; st < args.smax; ++st) {
            cA = __shfl_sync(0xffffffffu, cA, cA, G);
            cB = __shfl_sync(0xffffffffu, cB, cB, G);
          }
        }
        const uint32_t vAB = __shfl_sync(0xffffffffu, pack_lo16(cA, cB), 0, G);  // both roots, one shuffle
        const uint32_t xA = vAB & args.sl_xmask, xB = (vAB >> 16) & args.sl_xmask;
        if (xA >= args.sl_leafmin) {
          if (rA == mA) kA = xA;
          rA += 2 * NG;
          aA = rA < rows;
          wA = 0;
          if (aA) bA = base_of(rA);
        } else {
          wA = xA * args.sl_wmul;
        }
        if (xB >= args.sl_leafmin) {
          if (rB == mB) kB = xB;
          rB += 2 * NG;
          aB = rB < rows;
          wB = 0;
          if (aB) bB = base_of(rB);
        } else {
          wB = xB * args.sl_wmul;
        }
      } while (__any_sync(0xffffffffu, aA || aB));
      if (mA < rows) asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * mA), "r"(kA) : "memory");
      if (mB < rows) asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * mB), "r"(kB) : "memory");
    } else if constexpr (SR == 2 && SL == 1) {
      // Two record streams per group, self-loop codes (WinTable::sl_*).  Per
      // window step and stream: entry, feature, compare, one shift selecting
      // the successor code, ceil(log2 h) select-free shfl doublings, the
      // root broadcast and one mask; then (sl_step) the stream either moves
      // to the exit window (LEA) or, on a leaf, stores the code, steps to its
      // next record by a constant address increment and restarts at the root
      // window -- all predicated, no divergent branch.  An exhausted stream
      // re-walks its last record (re-storing the same code) until every
      // stream of the warp is done.
      static_assert(Rec<A, kTma>::kRowLocal, "self-loop streams: records inside one 128-byte row");
      const uint32_t a4 = 4u * (uint32_t)A;
      auto base_of = [&](uint32_t rr) {
        const uint32_t ra4 = rr * a4, rowb = ra4 & ~127u;
        return (tile + rowb) | (((rowb >> 3) & 0x70u) ^ (ra4 & 127u));
      };
      const uint32_t ng2 = 2u * NG, dl = 4u * ng2;
      const uint32_t rA = g, rB = g + NG;
      // label address of each stream's last record (a stream without
      // records is done from the start and stores beyond `rows` only)
      const uint32_t lg2 = (uint32_t)__ffs(ng2) - 1u;  // ng2 = 64 / G: a power of two
      const uint32_t kA = rA < rows ? (rows - rA - 1u) >> lg2 : 0u, kB = rB < rows ? (rows - rB - 1u) >> lg2 : 0u;
      uint32_t lA = lbuf + 4u * rA, lB = lbuf + 4u * rB;
      const uint32_t eLA = lA + dl * kA, eLB = lB + dl * kB;
      uint32_t dA = rA >= rows ? 1u : 0u, dB = rB >= rows ? 1u : 0u;
      uint32_t bA = base_of(rA < rows ? rA : 0u), bB = base_of(rB < rows ? rB : 0u);
      uint32_t aA = jaddr, aB = jaddr;
      // lane j of the group collects the code of its stream's j-th record in
      // a register (label address myA / myB): no shared-memory store per
      // resolution; one store per lane at the end of the slot
      const uint32_t myA = lbuf + 4u * (rA + ng2 * j), myB = myA + 4u * NG;
      uint32_t kcA = 0u, kcB = 0u;
      // one stream's terminal step (x = masked root code)
      auto sl_step = [&](uint32_t x, uint32_t& a, uint32_t& b, uint32_t& l, uint32_t& d, uint32_t& kc,
                         uint32_t el, uint32_t my) {
        asm volatile(
            "{\n\t"
            ".reg .pred lf, cap, adv, fin;\n\t"
            ".reg .u32 t;\n\t"
            "setp.ge.u32 lf, %5, %7;\n\t"
            "setp.eq.and.u32 cap, %2, %8, lf;\n\t"
            "@cap mov.u32 %4, %5;\n\t"
            "setp.ne.and.u32 adv, %2, %6, lf;\n\t"
            "setp.eq.and.u32 fin, %2, %6, lf;\n\t"
            "@adv add.u32 %2, %2, %9;\n\t"
            "@adv add.u32 %1, %1, %10;\n\t"
            "@adv xor.b32 %1, %1, %11;\n\t"
            "@fin mov.u32 %3, 1;\n\t"
            "mad.lo.u32 t, %5, %12, %13;\n\t"
            "selp.u32 %0, %13, t, lf;\n\t"
            "}"
            : "=r"(a), "+r"(b), "+r"(l), "+r"(d), "+r"(kc)
            : "r"(x), "r"(el), "r"(args.sl_leafmin), "r"(my), "r"(dl), "r"(args.sl_adv), "r"(args.sl_xor),
              "r"(args.sl_wmul), "r"(jaddr));
      };
      do {
        const uint2 eA = lds_u2(aA), eB = lds_u2(aB);
        const float vA = lds_f32((eA.y & args.cw_amask) ^ bA), vB = lds_f32((eB.y & args.cw_amask) ^ bB);
        uint32_t cA = eA.y >> (vA > __uint_as_float(eA.x) ? args.cw_rsh : args.cw_lsh);
        uint32_t cB = eB.y >> (vB > __uint_as_float(eB.x) ? args.cw_rsh : args.cw_lsh);
        if constexpr (STEPS >= 0) {
#pragma unroll
          for (int st = 0; st < STEPS; ++st) {
            cA = __shfl_sync(0xffffffffu, cA, cA, G);
            cB = __shfl_sync(0xffffffffu, cB, cB, G);
          }
        } else {
          for (uint32_t st = 0; st < args.smax; ++st) {
            cA = __shfl_sync(0xffffffffu, cA, cA, G);
            cB = __shfl_sync(0xffffffffu, cB, cB, G);
          }
        }
        const uint32_t vAB = __shfl_sync(0xffffffffu, pack_lo16(cA, cB), 0, G);  // both roots, one shuffle
        const uint32_t xA = vAB & args.sl_xmask, xB = (vAB >> 16) & args.sl_xmask;
        sl_step(xA, aA, bA, lA, dA, kcA, eLA, myA);
        sl_step(xB, aB, bB, lB, dB, kcB, eLB, myB);
      } while (__any_sync(0xffffffffu, (dA & dB) == 0u));
      if (rA + ng2 * j < rows) asm volatile("st.shared.u32 [%0], %1;" ::"r"(myA), "r"(kcA) : "memory");
      if (rB + ng2 * j < rows) asm volatile("st.shared.u32 [%0], %1;" ::"r"(myB), "r"(kcB) : "memory");
    } else if constexpr (SR == 2 && WIN_SHARED && Rec<A, kTma>::kRowLocal) {
      // Two record streams per group in the lean style (no predication; an
      // exhausted stream re-walks its last record): two independent window
      // chains per lane to overlap the entry -> feature -> shuffle latencies.
      const uint32_t a4 = 4u * (uint32_t)A;
      auto base_of = [&](uint32_t rr) {
        const uint32_t ra4 = rr * a4, rowb = ra4 & ~127u;
        return (tile + rowb) | (((rowb >> 3) & 0x70u) ^ (ra4 & 127u));
      };
      uint32_t rA = g, rB = g + NG;
      bool aA = rA < rows, aB = rB < rows;
      uint32_t wA = 0, wB = 0;
      uint32_t bA = base_of(aA ? rA : 0u), bB = base_of(aB ? rB : 0u);
      do {
        const Ent eA = load_ent(wA), eB = load_ent(wB);
        const float vA = lds_f32(ent_attr4(eA) ^ bA), vB = lds_f32(ent_attr4(eB) ^ bB);
        uint32_t cA = ent_next(eA, vA > __uint_as_float(eA.thr));
        uint32_t cB = ent_next(eB, vB > __uint_as_float(eB.thr));
        auto jump = [&]() {
          const uint32_t uA = __shfl_sync(0xffffffffu, cA, cA, G);
          const uint32_t uB = __shfl_sync(0xffffffffu, cB, cB, G);
          cA = (cA < 32u) ? uA : cA;
          cB = (cB < 32u) ? uB : cB;
        };
        if constexpr (STEPS >= 0) {
#pragma unroll
          for (int st = 0; st < STEPS; ++st) jump();
        } else {
          for (uint32_t st = 0; st < args.smax; ++st) jump();
        }
        const uint32_t rtA = __shfl_sync(0xffffffffu, cA, 0, G);
        const uint32_t rtB = __shfl_sync(0xffffffffu, cB, 0, G);
        if (rtA & leafbit) {
          if (aA && j == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * rA), "r"(rtA) : "memory");
          rA += 2 * NG;
          aA = rA < rows;
          wA = 0;
          if (aA) bA = base_of(rA);
        } else {
          wA = exit_off(rtA);
        }
        if (rtB & leafbit) {
          if (aB && j == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(lbuf + 4u * rB), "r"(rtB) : "memory");
          rB += 2 * NG;
          aB = rB < rows;
          wB = 0;
          if (aB) bB = base_of(rB);
        } else {
          wB = exit_off(rtB);
        }
      } while (__any_sync(0xffffffffu, aA || aB));
    } else {
      static_assert(SR >= 0 && SR <= 2, "one window, or one or two record streams per group");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the TMA refill
    __syncwarp();
    if constexpr (FR) {
      if (lane == 0) {  // refill now if the next tile's frame is out, else hand over deferred
        const uint32_t w = ((gen + 1u) << 1) | (fr_try_fill(tk + NS, b) ? 0u : 1u);
        asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(gen0 + 4u * b), "r"(w) : "memory");
      }
    } else if (tk + NS < my_tiles) {
      fill(tk + NS, b);  // this warp freed slot b: refill it ...
      if (lane == 0)  // ... and publish that generation tk / NS + 1 is on its way
        asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(gen0 + 4u * b), "r"(gen + 1u) : "memory");
    }
#pragma unroll
    for (int k = 0; k < (R + 31) / 32; ++k) {
      const uint32_t rr = lane + 32u * k;
      if (rr < rows) {
        uint32_t code;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(code) : "r"(lbuf + 4u * rr));
        const uint32_t cls = ((code & args.lab_mask) >> args.lab_shift) - args.lab_sub;
        labels[r0 + rr] = args.leaf_class ? __ldg(args.leaf_class + cls) : cls;
      }
    }
    __syncwarp();
  }
  if constexpr (FR) flush_count();
}

// ---------------------------------------------------------------------------
// K3: random forest with per-record majority vote
// ---------------------------------------------------------------------------
struct ForestArgs {
  PipeArgs p;
  const CNode* nodes;         // all trees, compact (child offsets relative to each tree)
  const uint32_t* offsets;    // t+1 node offsets
  uint32_t t_count, n_classes, abits;
  uint32_t* labels;
  uint32_t ns, stage_bytes;
};

// PACKED: n_classes <= 8 and t_count <= 255 -> two registers of 8-bit
// counters per record; otherwise per-warp shared counters.
template <int A, int LOADER, bool PACKED>
__global__ void __launch_bounds__(kMaxThreads)
    k_forest(const ForestArgs args, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int R = 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nw = blockDim.x >> 5;  // warps in this CTA
  const uint32_t sbase = align1024(smem_u32(smem));

  Pipe<A, 1, LOADER> pipe;
  pipe.tiles = sbase + (uint32_t)warp * args.ns * args.stage_bytes;
  pipe.bars = sbase + nw * args.ns * args.stage_bytes + (uint32_t)warp * args.ns * 8u;
  pipe.stride_bytes = args.stage_bytes;
  pipe.ns = args.ns;
  pipe.tmap = &tmap;
  pipe.p = args.p;
  pipe.lane = lane;
  const uint32_t counts = sbase + nw * args.ns * (args.stage_bytes + 8u) +
                          (uint32_t)warp * args.n_classes * 32u * 4u;

  const uint32_t amask = (1u << args.abits) - 1u;
  const uint64_t m = args.p.m;
  const uint64_t n_tiles = (m + R - 1) / R;
  const uint64_t step = (uint64_t)gridDim.x * nw;
  const uint64_t first = (uint64_t)blockIdx.x * nw + warp;
  pipe.start(first, step, n_tiles);

  uint64_t i = 0;
  for (uint64_t t = first; t < n_tiles; t += step, ++i) {
    const uint64_t r0 = t * (uint64_t)R;
    const uint32_t tile = pipe.acquire(i, t);
    const bool valid = r0 + lane < m;
    const uint32_t rr = valid ? lane : 0u;
    Rec<A, LOADER> rec;
    rec.init(tile, rr, args.p.a, args.p.x, r0 + rr, args.p.ld, args.p.layout_soa);
    uint32_t h0 = 0, h1 = 0;
    if constexpr (!PACKED)
      for (uint32_t c = 0; c < args.n_classes; ++c)
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(counts + (c * 32u + lane) * 4u), "r"(0u)
                     : "memory");
    for (uint32_t tr = 0; tr < args.t_count; ++tr) {
      const char* tn = reinterpret_cast<const char*>(args.nodes + __ldg(args.offsets + tr));
      uint2 nd = __ldg(reinterpret_cast<const uint2*>(tn));
      while (!(nd.y & kLeafBit)) {
        const float v = rec.get(nd.y & amask);
        nd = __ldg(reinterpret_cast<const uint2*>(
            tn + (nd.y >> args.abits) + (v > __uint_as_float(nd.x) ? 8u : 0u)));
      }
      uint32_t c = nd.y & ~kLeafBit;
      if (nd.y & kPairBit)  // folded terminal
        c = ((rec.get(nd.y & 0x3FFu) > __uint_as_float(nd.x)) ? (nd.y >> 20) : (nd.y >> 10)) & 0x3FFu;
      if constexpr (PACKED) {
        if (c < 4) h0 += 1u << (8 * c);
        else h1 += 1u << (8 * (c - 4));
      } else {
        const uint32_t a = counts + (c * 32u + lane) * 4u;
        uint32_t cur;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cur) : "r"(a));
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(cur + 1u) : "memory");
      }
    }
    // argmax, smallest class id wins ties
    uint32_t best = 0, bestc = 0;
    for (uint32_t c = 0; c < args.n_classes; ++c) {
      uint32_t cnt;
      if constexpr (PACKED) {
        cnt = ((c < 4 ? h0 : h1) >> (8 * (c & 3))) & 0xFFu;
      } else {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cnt) : "r"(counts + (c * 32u + lane) * 4u));
      }
      if (cnt > bestc) {
        bestc = cnt;
        best = c;
      }
    }
    if (valid) args.labels[r0 + lane] = best;
    pipe.release(i, t, step, n_tiles);
  }
}

// ---------------------------------------------------------------------------
// K3b: forest vote with trees streamed through shared memory
// ---------------------------------------------------------------------------
// Every warp keeps one TMA-staged tile of 32*S records resident for the whole
// tree loop; the CTA streams the T trees through a double buffer in shared
// memory (one elected thread issues cp.async.bulk for tree i+1 while all warps
// walk tree i; a CTA barrier per tree releases the buffer).  Votes live in
// packed 8-bit registers (<= 8 classes, <= 255 trees).
struct Forest2Args {
  PipeArgs p;
  const CNode* nodes;          // all trees, compact (child offsets relative to each tree)
  const uint32_t* offsets;     // t+1 node offsets (device)
  uint32_t t_count, n_classes, abits;
  uint32_t* labels;
  uint32_t stage_bytes;        // record tile (one stage per warp)
  uint32_t tree_buf_bytes;     // per tree buffer (>= largest tree, 16-aligned)
  uint32_t n_tree_bufs;        // tree ring depth (>= 2)
  uint32_t tree_region;        // bytes reserved for the ring (1024-aligned)
  const uint32_t* tree_bytes;  // per tree: bytes to copy (16-aligned, device)
};

// Warp-specialised: warp 0 is the tree producer (one elected lane issues
// cp.async.bulk into a ring of NT slots, gated by per-slot "empty" mbarriers
// that every consumer warp arrives on); warps 1..nw-1 are consumers that walk
// their resident record tile through each tree as soon as its "full" barrier
// flips -- consumers drift up to NT trees apart instead of meeting at a CTA
// barrier per tree.  Each consumer lane walks U trees at once (U independent
// dependent-load chains per lane: the walk is shared-memory-latency bound, so
// chains per SM, not warps, are what hide it; U trees cost tree-ring slots,
// which are cheaper than record tiles).

// One predicated level step of a forest walk over an attribute-major record
// tile: if the node is internal, node = tb + child + 8*(x[attr] > thr).
// Leaves are left untouched (no branch, no shared-memory traffic).
__device__ __forceinline__ void forest_step(uint32_t& thr, uint32_t& meta, uint32_t tb, uint32_t soa,
                                            uint32_t amask, uint32_t abits) {
  asm volatile(
      "{\n\t"
      ".reg .pred p, q;\n\t"
      ".reg .u32 fa, ch;\n\t"
      ".reg .f32 v;\n\t"
      "setp.ge.s32 p, %1, 0;\n\t"
      "and.b32 fa, %1, %4;\n\t"
      "shl.b32 fa, fa, 5;\n\t"
      "add.u32 fa, fa, %3;\n\t"
      "@p ld.shared.f32 v, [fa];\n\t"
      "setp.gt.and.f32 q, v, %0, p;\n\t"
      "shr.u32 ch, %1, %5;\n\t"
      "add.u32 ch, ch, %2;\n\t"
      "@q add.u32 ch, ch, 8;\n\t"
      "@p ld.shared.v2.u32 {%0, %1}, [ch];\n\t"
      "}"
      : "+f"(*reinterpret_cast<float*>(&thr)), "+r"(meta)
      : "r"(tb), "r"(soa), "r"(amask), "r"(abits)
      : "memory");
}

template <int A, int S, int U>
__global__ void __launch_bounds__(kForestMaxThreads)
    k_forest_smem(const Forest2Args args, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int R = 32 * S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nw = blockDim.x >> 5;
  const uint32_t nc = nw - 1;  // consumer warps
  const uint32_t sbase = align1024(smem_u32(smem));
  // [tree ring (1024-aligned)] [consumer stages] [consumer tile bars] [full bars] [empty bars]
  const uint32_t tbuf0 = sbase;
  const uint32_t tiles0 = sbase + args.tree_region;
  const uint32_t NT = args.n_tree_bufs;
  const uint32_t full0 = tiles0 + nc * (args.stage_bytes + 8u);
  const uint32_t empty0 = full0 + 8u * NT;
  const uint32_t T = args.t_count;

  const uint64_t m = args.p.m;
  const uint64_t n_tiles = (m + R - 1) / R;
  const uint64_t step = (uint64_t)gridDim.x * nc;
  const uint64_t base_tile = (uint64_t)blockIdx.x * nc;
  const uint64_t my_rounds = base_tile < n_tiles ? (n_tiles - base_tile + step - 1) / step : 0;
  const uint64_t total = my_rounds * T;  // trees this CTA streams

  if (threadIdx.x == 0) {
    for (uint32_t b = 0; b < NT; ++b) {
      mbar_init(full0 + 8u * b, 1);
      mbar_init(empty0 + 8u * b, nc);
    }
    fence_barrier_init();
  }
  Pipe<A, S, kTma> pipe;
  const uint32_t cw = warp > 0 ? (uint32_t)warp - 1 : 0u;
  pipe.tiles = tiles0 + cw * args.stage_bytes;
  pipe.bars = tiles0 + nc * args.stage_bytes + cw * 8u;
  pipe.stride_bytes = args.stage_bytes;
  pipe.ns = 1;
  pipe.tmap = &tmap;
  pipe.p = args.p;
  pipe.lane = lane;
  const uint64_t first = base_tile + cw;
  if (warp > 0) pipe.start(first, step, n_tiles);  // consumer tile barrier + first tile
  __syncthreads();

  if (warp == 0) {  // ---- producer -----------------------------------------
    if (lane == 0) {
      uint32_t b = 0, ph = 0, tr = 0;
      for (uint64_t gi = 0; gi < total; ++gi) {
        if (gi >= NT) {
          mbar_wait(empty0 + 8u * b, ph ^ 1u);
          // consumers' generic-proxy reads of the slot precede this async write
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const uint32_t bytes = __ldg(args.tree_bytes + tr);
        mbar_arrive_expect_tx(full0 + 8u * b, bytes);
        bulk_load(tbuf0 + b * args.tree_buf_bytes, args.nodes + __ldg(args.offsets + tr), bytes,
                  full0 + 8u * b);
        if (++tr == T) tr = 0;
        if (++b == NT) b = 0, ph ^= 1u;
      }
    }
    return;
  }

  // ---- consumers -----------------------------------------------------------
  const uint32_t amask = (1u << args.abits) - 1u;
  uint32_t b0 = 0, ph0 = 0;  // ring slot / phase of the next tree this warp consumes
  for (uint64_t k = 0; k < my_rounds; ++k) {
    const uint64_t t = first + k * step;
    const bool have = t < n_tiles;
    uint32_t tile = 0;
    if (have) tile = pipe.acquire(k, t);
    const uint64_t r0 = t * (uint64_t)R;
    Rec<A, kTma> rec[S];
    uint32_t h0[S], h1[S];
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const uint32_t r = q * 32 + lane;
      rec[q].init(tile, r, args.p.a, args.p.x, r0 + r, args.p.ld, 0);
      h0[q] = h1[q] = 0;
    }
    // Transpose the tile in place to attribute-major (feature (a, lane) at
    // tile + 4*(32a + lane)): every later feature read is bank-conflict free,
    // and the record is read by all T trees, so the one-off cost vanishes.
    constexpr bool kTranspose = (S == 1 && A > 0 && A <= 64);
    if constexpr (kTranspose) {
      if (have) {
        float v[A > 0 ? A : 1];
#pragma unroll
        for (int a = 0; a < A; ++a) v[a] = rec[0].get(4u * a);
        __syncwarp();
#pragma unroll
        for (int a = 0; a < A; ++a) sts_f32(tile + 4u * (32u * a + lane), v[a]);
        __syncwarp();
      }
    }
    const uint32_t soa = tile + 4u * lane;
    for (uint32_t tr = 0; tr < T; tr += U) {
      const uint32_t nu = min((uint32_t)U, T - tr);  // trees in this step
      uint32_t tb[U], thr[U], meta[U], slot[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        slot[u] = b0;
        tb[u] = tbuf0 + b0 * args.tree_buf_bytes;
        meta[u] = kLeafBit;
        thr[u] = 0;
        if ((uint32_t)u < nu) {
          mbar_wait(full0 + 8u * b0, ph0);
          if (++b0 == NT) b0 = 0, ph0 ^= 1u;
        }
      }
      if (have) {
        if constexpr (kTranspose) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if ((uint32_t)u < nu) {
              const uint2 n = lds_u2(tb[u]);
              thr[u] = n.x;
              meta[u] = n.y;
            }
          }
          // U predicated chains per lane until every chain sits on a leaf
          while (true) {
            bool any = false;
#pragma unroll
            for (int u = 0; u < U; ++u) any |= (int)meta[u] >= 0;
            if (!any) break;
#pragma unroll
            for (int u = 0; u < U; ++u) forest_step(thr[u], meta[u], tb[u], soa, amask, args.abits);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {  // folded terminal: the last predicate picks the pair's leaf
            if (meta[u] & kPairBit) {
              const float v = lds_f32(soa + ((meta[u] & 0x3FFu) << 5));
              const uint32_t c = (v > __uint_as_float(thr[u])) ? (meta[u] >> 20) : (meta[u] >> 10);
              meta[u] = kLeafBit | (c & 0x3FFu);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if ((uint32_t)u < nu) {
              const uint32_t c = meta[u] & ~kLeafBit;
              if (c < 4) h0[0] += 1u << (8 * c);
              else h1[0] += 1u << (8 * (c - 4));
            }
          }
        } else {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if ((uint32_t)u >= nu) continue;
#pragma unroll
            for (int q = 0; q < S; ++q) {
              uint2 nd = lds_u2(tb[u]);
              while (!(nd.y & kLeafBit)) {
                const float v = rec[q].get(nd.y & amask);
                nd = lds_u2(tb[u] + (nd.y >> args.abits) + (v > __uint_as_float(nd.x) ? 8u : 0u));
              }
              uint32_t c = nd.y & ~kLeafBit;
              if (nd.y & kPairBit)
                c = ((rec[q].get(nd.y & 0x3FFu) > __uint_as_float(nd.x)) ? (nd.y >> 20) : (nd.y >> 10)) & 0x3FFu;
              if (c < 4) h0[q] += 1u << (8 * c);
              else h1[q] += 1u << (8 * (c - 4));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if ((uint32_t)u < nu) mbar_arrive(empty0 + 8u * slot[u]);  // this warp is done with the slot
      }
    }
    if (have) {
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint64_t r = r0 + q * 32 + lane;
        uint32_t best = 0, bestc = 0;
        for (uint32_t c = 0; c < args.n_classes; ++c) {
          const uint32_t cnt = ((c < 4 ? h0[q] : h1[q]) >> (8 * (c & 3))) & 0xFFu;
          if (cnt > bestc) {
            bestc = cnt;
            best = c;
          }
        }
        if (r < m) args.labels[r] = best;
      }
      pipe.release(k, t, step, n_tiles);
    }
  }
}

// ---------------------------------------------------------------------------
// K2x: exact whole-tree speculation at CTA scope (reference counters for any I)
// ---------------------------------------------------------------------------
// The paper's Proc. 5 as written and the reference's
// mapped barrier-separated GroupWorker (eval_speculative.cpp:127-204): the CTA
// is one record group; thread j owns internal nodes map[j], map[j+T], ...;
// the path array is double-buffered in shared memory and every doubling is a
// barrier-separated snapshot step; while the root entry is internal, k
// doublings per iteration.  Leaves stay identity fixpoints in both buffers.
// Used when per-record counters are requested for trees whose internal nodes
// exceed one warp (the shfl kernel covers <= 32).
struct SpecExactArgs {
  PipeArgs p;
  const uint4* nodes;      // original 16-byte nodes
  const uint32_t* map;     // internal node indices ascending (processor_node_map)
  uint32_t n, I, k;
  uint32_t* labels;
  uint32_t* iters;
  uint32_t* steps;
  uint32_t* gbuf;          // null: path buffers in shared memory; else 2n + 1 words per CTA
                           // in global memory (trees whose two path arrays exceed shared memory)
};

template <int = 0>  // a template so every translation unit may include this header
__global__ void __launch_bounds__(kMaxThreads) k_spec_exact_cta(const SpecExactArgs args) {
  extern __shared__ __align__(1024) unsigned char smem[];
  uint32_t* buf_a = args.gbuf ? args.gbuf + (uint64_t)blockIdx.x * (2ull * args.n + 1)
                              : reinterpret_cast<uint32_t*>(smem);
  uint32_t* buf_b = buf_a + args.n;
  uint32_t& root_val = buf_b[args.n];  // dynamic smem only: opt-in size stays valid
  for (uint32_t i = threadIdx.x; i < args.n; i += blockDim.x) buf_a[i] = buf_b[i] = i;
  __syncthreads();
  for (uint64_t r = blockIdx.x; r < args.p.m; r += gridDim.x) {
    const float* rec = args.p.layout_soa ? args.p.x + r : args.p.x + r * (uint64_t)args.p.ld;
    const uint64_t astride = args.p.layout_soa ? args.p.ld : 1;
    uint32_t* cur = buf_a;
    uint32_t* alt = buf_b;
    // node evaluation over the mapped (internal) lanes
    for (uint32_t j = threadIdx.x; j < args.I; j += blockDim.x) {
      const uint32_t i = __ldg(args.map + j);
      const uint4 nd = __ldg(args.nodes + i);
      cur[i] = nd.z + (uint32_t)(__ldg(rec + (uint64_t)nd.x * astride) > __uint_as_float(nd.y));
    }
    __syncthreads();
    uint32_t it = 0, st = 0;
    while (true) {
      if (threadIdx.x == 0) root_val = __ldg(args.nodes + cur[0]).w;
      __syncthreads();
      const bool resolved = root_val != kNoClass;
      __syncthreads();
      if (resolved) break;
      for (uint32_t s = 0; s < args.k; ++s) {
        for (uint32_t j = threadIdx.x; j < args.I; j += blockDim.x) {
          const uint32_t i = __ldg(args.map + j);
          alt[i] = cur[cur[i]];
        }
        __syncthreads();
        uint32_t* t = cur;
        cur = alt;
        alt = t;
        ++st;
      }
      ++it;
    }
    if (threadIdx.x == 0) {
      args.labels[r] = __ldg(args.nodes + cur[0]).w;
      if (args.iters) {
        args.iters[r] = it;
        args.steps[r] = st;
      }
    }
    // an odd number of swaps left the live array in buf_b: no reset is
    // needed (every mapped entry is rewritten before it is read), but both
    // buffers must stop being read before the next record writes them
    __syncthreads();
  }
}

}  // namespace stk

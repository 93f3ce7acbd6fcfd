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
// All three share the record-tile stager: each warp streams tiles of 32*S
// records HBM -> registers (coalesced 128-bit ld.global.nc, one tile of
// prefetch in flight while the previous tile is walked) -> a per-warp shared
// memory tile whose word-level XOR swizzle makes both the staging stores and
// "all lanes read the same attribute" (every root visit) bank-conflict free.
//
// Semantics (bit-exact with the reference): successor = child + (x > thr)
// with an ordered IEEE compare and no flush-to-zero (tree.hpp:51-54); build
// without --use_fast_math / -ftz=true.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace stk {

constexpr uint32_t kLeafBit = 0x80000000u;  // compact-node meta: leaf marker
constexpr uint32_t kExitBit = 0x40000000u;  // speculative code: exit to window
constexpr uint32_t kNoClass = 0xFFFFFFFFu;
constexpr int kWarpsPerCta = 8;

// Compact 8-byte device node.  internal: meta = child << abits | attr (bit 31
// clear); leaf: meta = kLeafBit | class (or | leaf ordinal when a class does
// not fit in 31 bits; the host then passes a leaf-class table).
struct __align__(8) CNode {
  float thr;
  uint32_t meta;
};

// Speculative window entry (16 B): lane j of a window evaluates one internal
// node.  y = attr | steps << 24 (steps = doubling count that resolves this
// window); z/w = left/right successor codes: < 32 lane index inside the
// window, kExitBit | base of the next window, or kLeafBit | class/ordinal.
struct __align__(16) SEntry {
  float thr;
  uint32_t attr_steps;
  uint32_t left;
  uint32_t right;
};

enum Loader { kVec = 0, kScalar = 1, kSoa = 2, kDirect = 3 };
enum TreeLoc { kShared = 1, kConst = 2, kGlobal = 3, kWide = 4 };

// ---------------------------------------------------------------------------
// Tile geometry.  A > 0: compile-time arity; A == 0: runtime arity.
// ---------------------------------------------------------------------------
template <int A>
struct TileGeom {
  static constexpr bool kPow2Small = A > 0 && (A & (A - 1)) == 0 && A <= 32;
  static constexpr bool kMult32 = A > 0 && (A % 32) == 0;
  static constexpr int kLog2 = A == 1 ? 0 : A == 2 ? 1 : A == 4 ? 2 : A == 8 ? 3 : A == 16 ? 4 : 5;
  // row pitch in words
  static __host__ __device__ __forceinline__ uint32_t pitch(uint32_t a_rt) {
    if constexpr (kPow2Small || kMult32) return (uint32_t)A;
    else if constexpr (A > 0) return (A & 1) ? A : A + 1;
    else return a_rt | 1u;
  }
  // word offset of (row r, attribute a) inside a tile
  static __device__ __forceinline__ uint32_t addr(uint32_t r, uint32_t a, uint32_t p) {
    if constexpr (kPow2Small) {
      return r * A + (a ^ ((r >> (5 - kLog2)) & (A - 1)));
    } else if constexpr (kMult32) {
      const uint32_t g = r * (A / 32) + (a >> 5);
      return r * A + (a & ~31u) + ((a & 31u) ^ ((g + (g >> 5)) & 31u));
    } else {
      return r * p + a;
    }
  }
};

// Streaming 128-bit read-only load that does not allocate in L1.
__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// ---------------------------------------------------------------------------
// Per-warp tile stager.  Tile t covers records [t*R, t*R + R), R = 32*S.
// ---------------------------------------------------------------------------
template <int A, int S, int LOADER>
struct Stager {
  static constexpr int R = 32 * S;
  // float4 per lane for a full vector tile (A compile-time only)
  static constexpr int V = A > 0 ? (R * A / 4 + 31) / 32 : 1;
  float4 buf[LOADER == kVec ? V : 1];

  const float* __restrict__ x;
  uint64_t m;
  uint32_t a, ld, p;

  __device__ __forceinline__ bool full(uint64_t t) const { return (t + 1) * (uint64_t)R <= m; }

  // Issue the global loads of tile t into registers (vector path, full tiles).
  __device__ __forceinline__ void prefetch(uint64_t t, int lane) {
    if constexpr (LOADER == kVec) {
      if (full(t)) {
        const float4* src = reinterpret_cast<const float4*>(x + t * (uint64_t)R * A);
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const int f4 = lane + 32 * k;
          if ((R * A / 4) % 32 == 0 || f4 < R * A / 4) buf[k] = ld_stream(src + f4);
        }
      }
    }
  }

  // Write tile t into the shared tile `s` (after prefetch for the vector path).
  __device__ __forceinline__ void commit(uint64_t t, float* __restrict__ s, int lane) {
    using Gm = TileGeom<A>;
    if constexpr (LOADER == kVec) {
      if (full(t)) {
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const int f4 = lane + 32 * k;
          if ((R * A / 4) % 32 == 0 || f4 < R * A / 4) {
            const float vals[4] = {buf[k].x, buf[k].y, buf[k].z, buf[k].w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t f = 4u * f4 + c;
              const uint32_t r = f / A, aa = f % A;
              s[Gm::addr(r, aa, p)] = vals[c];
            }
          }
        }
        return;
      }
    }
    if constexpr (LOADER == kSoa) {
      // x[attr * ld + record]: one coalesced 128 B load per attribute and lane-row
      const uint64_t r0 = t * (uint64_t)R;
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint32_t r = q * 32 + lane;
        const bool ok = r0 + r < m;
        for (uint32_t aa = 0; aa < a; ++aa)
          s[Gm::addr(r, aa, p)] = ok ? __ldg(x + (uint64_t)aa * ld + r0 + r) : 0.0f;
      }
      return;
    }
    // scalar AoS path (runtime arity / strided rows / the partial last tile)
    {
      const uint64_t r0 = t * (uint64_t)R;
      const uint32_t rows = (uint32_t)((m - r0) < (uint64_t)R ? (m - r0) : (uint64_t)R);
      const uint32_t total = rows * a;
      if (ld == a) {
        const float* src = x + r0 * a;
        for (uint32_t f = lane; f < total; f += 32) {
          const uint32_t r = f / a, aa = f - r * a;
          s[Gm::addr(r, aa, p)] = __ldg(src + f);
        }
      } else {
        for (uint32_t f = lane; f < total; f += 32) {
          const uint32_t r = f / a, aa = f - r * a;
          s[Gm::addr(r, aa, p)] = __ldg(x + (r0 + r) * (uint64_t)ld + aa);
        }
      }
    }
  }
};

// Feature accessor for one record inside the staged tile (or in global
// memory for the direct loader).
template <int A, int LOADER>
struct Feat {
  const float* __restrict__ base;  // tile (shared) or record row (global)
  uint32_t r, p;
  __device__ __forceinline__ float operator()(uint32_t a) const {
    if constexpr (LOADER == kDirect) return __ldg(base + a);
    else return base[TileGeom<A>::addr(r, a, p)];
  }
};

// ---------------------------------------------------------------------------
// Tree access
// ---------------------------------------------------------------------------
template <int CAP>
struct ConstTree {
  CNode n[CAP];
};

template <int TLOC, int CAP>
struct TreeRef {
  const CNode* __restrict__ s;  // shared or global compact nodes
  const ConstTree<CAP>* c;      // constant-bank copy
  __device__ __forceinline__ CNode get(uint32_t i) const {
    if constexpr (TLOC == kConst) return c->n[i];
    else if constexpr (TLOC == kGlobal) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(s) + i);
      return CNode{__uint_as_float(v.x), v.y};
    } else {
      return s[i];
    }
  }
};

struct DataArgs {
  const float* x;
  uint64_t m;
  uint32_t a, ld;
  const CNode* nodes;          // compact nodes (device global)
  const uint4* wide;           // original 16-byte nodes (kWide)
  uint32_t n_nodes;
  uint32_t abits;              // attr field width in compact meta
  const uint32_t* leaf_class;  // null: leaf meta carries the class
  uint32_t* labels;
};

// ---------------------------------------------------------------------------
// K1: data decomposition
// ---------------------------------------------------------------------------
template <int A, int S, int TLOC, int LOADER, int CAP>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    k_data(const DataArgs args, const __grid_constant__ ConstTree<CAP> ctree) {
  extern __shared__ __align__(16) unsigned char smem[];
  using Gm = TileGeom<A>;
  constexpr int R = 32 * S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t p = Gm::pitch(args.a);

  // ---- stage the node array once per CTA --------------------------------
  const CNode* tree_s = args.nodes;
  size_t tree_bytes = 0;
  if constexpr (TLOC == kShared) {
    tree_bytes = ((size_t)args.n_nodes * sizeof(CNode) + 15) & ~size_t(15);
    const uint4* src = reinterpret_cast<const uint4*>(args.nodes);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    const uint32_t n16 = (uint32_t)(tree_bytes / 16);
    for (uint32_t i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = __ldg(src + i);
    tree_s = reinterpret_cast<const CNode*>(smem);
    __syncthreads();
  }
  TreeRef<TLOC, CAP> tree{tree_s, &ctree};
  float* tile = reinterpret_cast<float*>(smem + tree_bytes) + (size_t)warp * R * p;

  Stager<A, S, LOADER> st;
  st.x = args.x;
  st.m = args.m;
  st.a = args.a;
  st.ld = args.ld;
  st.p = p;

  const uint64_t n_tiles = (args.m + R - 1) / R;
  const uint64_t wstride = (uint64_t)gridDim.x * kWarpsPerCta;
  uint64_t t = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  if (LOADER != kDirect && t < n_tiles) st.prefetch(t, lane);
  const uint32_t amask = (1u << args.abits) - 1u;

  for (; t < n_tiles; t += wstride) {
    const uint64_t r0 = t * (uint64_t)R;
    if constexpr (LOADER != kDirect) {
      __syncwarp();
      st.commit(t, tile, lane);
      __syncwarp();
      if (t + wstride < n_tiles) st.prefetch(t + wstride, lane);
    }
    if constexpr (TLOC == kWide) {
      // generic 16-byte node path: the reference loop verbatim
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint32_t r = q * 32 + lane;
        Feat<A, LOADER> f{LOADER == kDirect ? args.x + (r0 + r) * (uint64_t)args.ld : tile, r, p};
        if (r0 + r >= args.m) continue;
        uint32_t i = 0;
        uint4 nd = __ldg(args.wide);
        while (nd.w == kNoClass) {
          i = nd.z + (uint32_t)(f(nd.x) > __uint_as_float(nd.y));
          nd = __ldg(args.wide + i);
        }
        args.labels[r0 + r] = nd.w;
      }
    } else {
      float thr[S];
      uint32_t meta[S];
      const CNode root = tree.get(0);
#pragma unroll
      for (int q = 0; q < S; ++q) {
        thr[q] = root.thr;
        meta[q] = root.meta;
        if (r0 + q * 32 + lane >= args.m) meta[q] = kLeafBit;  // idle lane-slot
      }
      // Branch-free successor per level; a lane leaves the loop once all its
      // S walks sit on leaves (warp pays its slowest record per tile).
      while (true) {
        bool any = false;
#pragma unroll
        for (int q = 0; q < S; ++q) {
          if (!(meta[q] & kLeafBit)) {
            const uint32_t r = q * 32 + lane;
            Feat<A, LOADER> f{LOADER == kDirect ? args.x + (r0 + r) * (uint64_t)args.ld : tile, r, p};
            const float v = f(meta[q] & amask);
            const uint32_t i = (meta[q] >> args.abits) + (uint32_t)(v > thr[q]);
            const CNode nd = tree.get(i);
            thr[q] = nd.thr;
            meta[q] = nd.meta;
            any = true;
          }
        }
        if (!any) break;
      }
#pragma unroll
      for (int q = 0; q < S; ++q) {
        const uint64_t r = r0 + q * 32 + lane;
        if (r < args.m) {
          const uint32_t c = meta[q] & ~kLeafBit;
          args.labels[r] = args.leaf_class ? __ldg(args.leaf_class + c) : c;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K2: speculative decomposition with shfl pointer-jumping
// ---------------------------------------------------------------------------
struct SpecArgs {
  const float* x;
  uint64_t m;
  uint32_t a, ld;
  const SEntry* win;     // window table (device global), padded by 32 entries
  uint32_t n_entries;    // incl. padding
  uint32_t root_code;    // code of the root: kExitBit|0, or kLeafBit|class for N == 1
  uint32_t G;            // lanes per record group (power of two <= 32)
  uint32_t k;            // 0: fixed per-window steps; >=1: check root every k steps
  const uint32_t* leaf_class;
  uint32_t* labels;
  uint32_t* iters;       // nullable per-record counters
  uint32_t* steps;
};

template <int A, int LOADER, bool WIN_SHARED>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_spec(const SpecArgs args) {
  extern __shared__ __align__(16) unsigned char smem[];
  using Gm = TileGeom<A>;
  constexpr int R = 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t p = Gm::pitch(args.a);

  const SEntry* win = args.win;
  size_t win_bytes = 0;
  if constexpr (WIN_SHARED) {
    win_bytes = (size_t)args.n_entries * sizeof(SEntry);
    const uint4* src = reinterpret_cast<const uint4*>(args.win);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (uint32_t i = threadIdx.x; i < args.n_entries; i += blockDim.x) dst[i] = __ldg(src + i);
    win = reinterpret_cast<const SEntry*>(smem);
    __syncthreads();
  }
  float* tile = reinterpret_cast<float*>(smem + win_bytes) + (size_t)warp * R * p;

  Stager<A, 1, LOADER> st;
  st.x = args.x;
  st.m = args.m;
  st.a = args.a;
  st.ld = args.ld;
  st.p = p;

  const uint32_t G = args.G;
  const uint32_t NG = 32u / G;       // record groups per warp
  const uint32_t g = lane / G;       // my group
  const uint32_t j = lane & (G - 1); // my lane in the group = window-local node
  const uint32_t gbase = g * G;
  const bool counting = args.iters != nullptr;

  const uint64_t n_tiles = (args.m + R - 1) / R;
  const uint64_t wstride = (uint64_t)gridDim.x * kWarpsPerCta;
  uint64_t t = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  if (LOADER != kDirect && t < n_tiles) st.prefetch(t, lane);

  for (; t < n_tiles; t += wstride) {
    const uint64_t r0 = t * (uint64_t)R;
    if constexpr (LOADER != kDirect) {
      __syncwarp();
      st.commit(t, tile, lane);
      __syncwarp();
      if (t + wstride < n_tiles) st.prefetch(t + wstride, lane);
    }
    const uint32_t rows = (uint32_t)((args.m - r0) < (uint64_t)R ? (args.m - r0) : (uint64_t)R);
    // Group g classifies tile rows g, g+NG, ...; a finished group refills
    // with its next row immediately, so skewed depths do not idle it.
    uint32_t r = g;
    uint32_t code = args.root_code;  // current window (exit code) or leaf
    bool active = r < rows;
    uint32_t n_it = 0, n_st = 0;
    while (__any_sync(0xffffffffu, active)) {
      const uint32_t rr = active ? r : 0u;
      const uint32_t base = code & ~(kExitBit | kLeafBit);
      const bool evaluating = active && !(code & kLeafBit);
      // -- node evaluation: every window lane computes its successor --------
      const SEntry e = win[(evaluating ? base : 0u) + j];
      Feat<A, LOADER> f{LOADER == kDirect ? args.x + (r0 + rr) * (uint64_t)args.ld : tile, rr, p};
      const float v = f(e.attr_steps & 0x00FFFFFFu);
      uint32_t c = (v > e.thr) ? e.right : e.left;
      // -- path reduction: shfl pointer-jumping inside the group ------------
      const uint32_t wsteps = __shfl_sync(0xffffffffu, e.attr_steps >> 24, gbase);
      if (args.k == 0) {
        const uint32_t smax = __reduce_max_sync(0xffffffffu, evaluating ? wsteps : 0u);
        for (uint32_t s = 0; s < smax; ++s) {
          const uint32_t u = __shfl_sync(0xffffffffu, c, c & (G - 1), G);
          if (c < 32u) c = u;
        }
        if (counting && evaluating) {
          n_it += 1;
          n_st += wsteps;
        }
      } else {
        // reference barrier_separated loop: while root unresolved, k doublings
        while (true) {
          const uint32_t root = __shfl_sync(0xffffffffu, c, gbase);
          const bool need = evaluating && root < 32u;
          if (!__any_sync(0xffffffffu, need)) break;
          for (uint32_t s = 0; s < args.k; ++s) {
            const uint32_t u = __shfl_sync(0xffffffffu, c, c & (G - 1), G);
            if (need && c < 32u) c = u;
          }
          if (need) {
            n_it += 1;
            n_st += args.k;
          }
        }
      }
      const uint32_t root = __shfl_sync(0xffffffffu, c, gbase);
      if (active) {
        const uint32_t next = evaluating ? root : code;
        if (next & kLeafBit) {
          if (j == 0) {
            const uint32_t cls = next & ~kLeafBit;
            const uint64_t out = r0 + r;
            args.labels[out] = args.leaf_class ? __ldg(args.leaf_class + cls) : cls;
            if (counting) {
              args.iters[out] = n_it;
              args.steps[out] = n_st;
            }
          }
          n_it = n_st = 0;
          r += NG;
          code = args.root_code;
          active = r < rows;
        } else {
          code = next;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K3: random forest with per-record majority vote
// ---------------------------------------------------------------------------
struct ForestArgs {
  const float* x;
  uint64_t m;
  uint32_t a, ld;
  const CNode* nodes;         // all trees, compact
  const uint32_t* offsets;    // t+1 node offsets
  uint32_t t_count, n_classes, abits;
  uint32_t* labels;
};

// PACKED: n_classes <= 8 and t_count <= 255 -> two registers of 8-bit
// counters per record; otherwise per-warp shared counters.
template <int A, int LOADER, bool PACKED>
__global__ void __launch_bounds__(kWarpsPerCta * 32) k_forest(const ForestArgs args) {
  extern __shared__ __align__(16) unsigned char smem[];
  using Gm = TileGeom<A>;
  constexpr int R = 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t p = Gm::pitch(args.a);
  float* tile = reinterpret_cast<float*>(smem) + (size_t)warp * R * p;
  uint32_t* counts = reinterpret_cast<uint32_t*>(reinterpret_cast<float*>(smem) +
                                                 (size_t)kWarpsPerCta * R * p) +
                     (size_t)warp * args.n_classes * 32;

  Stager<A, 1, LOADER> st;
  st.x = args.x;
  st.m = args.m;
  st.a = args.a;
  st.ld = args.ld;
  st.p = p;
  const uint32_t amask = (1u << args.abits) - 1u;
  const uint64_t n_tiles = (args.m + R - 1) / R;
  const uint64_t wstride = (uint64_t)gridDim.x * kWarpsPerCta;
  uint64_t t = (uint64_t)blockIdx.x * kWarpsPerCta + warp;
  if (LOADER != kDirect && t < n_tiles) st.prefetch(t, lane);

  for (; t < n_tiles; t += wstride) {
    const uint64_t r0 = t * (uint64_t)R;
    if constexpr (LOADER != kDirect) {
      __syncwarp();
      st.commit(t, tile, lane);
      __syncwarp();
      if (t + wstride < n_tiles) st.prefetch(t + wstride, lane);
    }
    const bool valid = r0 + lane < args.m;
    const uint32_t rr = valid ? lane : 0u;
    Feat<A, LOADER> f{LOADER == kDirect ? args.x + (r0 + rr) * (uint64_t)args.ld : tile, rr, p};
    uint32_t h0 = 0, h1 = 0;
    if constexpr (!PACKED)
      for (uint32_t c = 0; c < args.n_classes; ++c) counts[c * 32 + lane] = 0;
    for (uint32_t tr = 0; tr < args.t_count; ++tr) {
      const uint2* tn = reinterpret_cast<const uint2*>(args.nodes + __ldg(args.offsets + tr));
      uint2 nd = __ldg(tn);
      while (!(nd.y & kLeafBit)) {
        const float v = f(nd.y & amask);
        nd = __ldg(tn + (nd.y >> args.abits) + (uint32_t)(v > __uint_as_float(nd.x)));
      }
      const uint32_t c = nd.y & ~kLeafBit;
      if constexpr (PACKED) {
        if (c < 4) h0 += 1u << (8 * c);
        else h1 += 1u << (8 * (c - 4));
      } else {
        counts[c * 32 + lane] += 1;
      }
    }
    // argmax, smallest class id wins ties
    uint32_t best = 0, bestc = 0;
    for (uint32_t c = 0; c < args.n_classes; ++c) {
      uint32_t cnt;
      if constexpr (PACKED) cnt = ((c < 4 ? h0 : h1) >> (8 * (c & 3))) & 0xFFu;
      else cnt = counts[c * 32 + lane];
      if (cnt > bestc) {
        bestc = cnt;
        best = c;
      }
    }
    if (valid) args.labels[r0 + lane] = best;
  }
}

}  // namespace stk

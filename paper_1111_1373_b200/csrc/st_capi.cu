// C-ABI implementation of include/spectree_b200.h.
//
// Host-side responsibilities (native C++, no Python on the path):
//   * tree preprocessing: validation (subset of tree.cpp:138-189), the compact
//     8-byte node format for the data kernel, the speculative window tables
//     (the paper's proposed level windows);
//   * lazy per-device replicas of every tree/forest (tree replicated to each
//     GPU);
//   * dispatch to the sm_100a kernels in st_kernels.cuh with an
//     occupancy-derived persistent grid;
//   * the host-buffer path (chunked H2D / kernel / D2H over two streams) and
//     the sample-sharded multi-GPU driver.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/spectree_b200.h"
#include "st_kernels.cuh"

using namespace stk;

static_assert(sizeof(st_node) == 16, "st_node must match spectree::EncodedNode");
static_assert(offsetof(st_node, attribute) == 0 && offsetof(st_node, threshold) == 4 &&
                  offsetof(st_node, child) == 8 && offsetof(st_node, class_id) == 12,
              "st_node field offsets must match spectree::EncodedNode");

namespace {

thread_local std::string g_error;
thread_local uint32_t g_launches = 0;

struct StError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, std::string msg) { throw StError{code, std::move(msg)}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
      fail(ST_ERR_NO_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
    std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
    if (e == cudaErrorMemoryAllocation) {
      size_t fr = 0, tot = 0;
      if (cudaMemGetInfo(&fr, &tot) == cudaSuccess)
        msg += " (device free " + std::to_string(fr >> 20) + " MiB of " + std::to_string(tot >> 20) + ")";
      cudaGetLastError();
    }
    fail(ST_ERR_CUDA, msg);
  }
}
#define CK(x) cuda_check((x), #x)

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_error.clear();
    return ST_OK;
  } catch (const StError& e) {
    g_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_error = "host allocation failed";
    return ST_ERR_CUDA;
  } catch (const std::exception& e) {
    g_error = e.what();
    return ST_ERR_CUDA;
  }
}

uint32_t ceil_log2(uint32_t v) {
  uint32_t s = 0, reach = 1;
  while (reach < v) {
    reach *= 2;
    ++s;
  }
  return s;
}

int current_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) fail(ST_ERR_NO_DEVICE, "no CUDA device available (no CPU fallback)");
  int d = 0;
  CK(cudaGetDevice(&d));
  return d;
}

struct DevProps {
  int sms = 0;
  size_t smem_optin = 0;
  size_t smem_per_sm = 0;
};
DevProps dev_props(int dev) {
  static std::mutex mu;
  static std::map<int, DevProps> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  DevProps p;
  int v = 0;
  CK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  p.sms = v;
  CK(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  p.smem_optin = (size_t)v;
  CK(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  p.smem_per_sm = (size_t)v;
  cache[dev] = p;
  return p;
}

// ---------------------------------------------------------------------------
// Speculative windows
// ---------------------------------------------------------------------------
struct WinTable {
  std::vector<SEntry> entries;  // padded by 32 entries
  uint32_t root_code = 0;
  uint32_t windows = 0;
  uint32_t max_steps = 0;
};

}  // namespace

namespace st_internal {
void set_error(const std::string& msg) { g_error = msg; }
void set_launches(uint32_t n) { g_launches = n; }
}  // namespace st_internal

struct st_tree {
  std::vector<st_node> nodes;
  st_tree_info info{};
  uint32_t abits = 1;
  bool compact_ok = true;
  bool leaf_table = false;            // some class >= 2^31: leaves carry ordinals
  std::vector<uint32_t> leaf_classes;  // ordinal -> class
  std::vector<uint32_t> leaf_code;     // node -> code payload (class or ordinal)
  std::vector<CNode> compact;

  std::mutex mu;
  std::map<std::pair<uint32_t, uint32_t>, std::shared_ptr<WinTable>> wins;  // (G, H)
  struct Dev {
    CNode* compact = nullptr;
    uint4* wide = nullptr;
    uint32_t* leaf_tbl = nullptr;
    uint32_t* internal_map = nullptr;  // processor_node_map (tree.cpp:204-209)
    std::map<std::pair<uint32_t, uint32_t>, SEntry*> wins;
  };
  std::map<int, Dev> dev;

  ~st_tree() {
    int cur = -1;
    cudaGetDevice(&cur);
    for (auto& kv : dev) {
      if (cudaSetDevice(kv.first) != cudaSuccess) continue;
      cudaFree(kv.second.compact);
      cudaFree(kv.second.wide);
      cudaFree(kv.second.leaf_tbl);
      cudaFree(kv.second.internal_map);
      for (auto& w : kv.second.wins) cudaFree(w.second);
    }
    if (cur >= 0) cudaSetDevice(cur);
  }

  bool is_leaf(uint32_t i) const { return nodes[i].class_id != ST_NO_CLASS; }

  std::shared_ptr<WinTable> windows(uint32_t G, uint32_t H) {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(G, H);
    auto it = wins.find(key);
    if (it != wins.end()) return it->second;
    auto w = std::make_shared<WinTable>(build_windows(G, H));
    wins[key] = w;
    return w;
  }

  // Partition the internal nodes into windows of <= G nodes and <= H levels,
  // breadth-first from each window root.  Lane j of a window holds its j-th
  // member (for a tree with I <= G internal nodes and H >= depth this is the
  // reference's processor_node_map, tree.cpp:204-209).
  WinTable build_windows(uint32_t G, uint32_t H) const {
    WinTable wt;
    const uint32_t n = (uint32_t)nodes.size();
    if (is_leaf(0)) {
      wt.root_code = kLeafBit | leaf_code[0];
      wt.entries.assign(32, SEntry{0.0f, 0u, 0u, 0u});
      return wt;
    }
    std::vector<int32_t> win_of_root(n, -1);
    std::vector<std::vector<uint32_t>> members;
    std::vector<std::vector<uint32_t>> ldepth;
    std::deque<uint32_t> roots;
    win_of_root[0] = 0;
    members.emplace_back();
    ldepth.emplace_back();
    roots.push_back(0);
    while (!roots.empty()) {
      const uint32_t root = roots.front();
      roots.pop_front();
      const int32_t w = win_of_root[root];
      std::vector<uint32_t> mem, dep;
      std::deque<std::pair<uint32_t, uint32_t>> q;
      q.emplace_back(root, 0);
      std::vector<std::pair<uint32_t, uint32_t>> exits;
      std::vector<uint32_t> seen;  // DAG-shaped inputs may reach a node twice
      while (!q.empty()) {
        auto [u, d] = q.front();
        q.pop_front();
        if (std::find(seen.begin(), seen.end(), u) != seen.end()) continue;
        seen.push_back(u);
        if (mem.size() >= G || d >= H) {
          exits.emplace_back(u, d);
          continue;
        }
        mem.push_back(u);
        dep.push_back(d);
        for (uint32_t c : {nodes[u].child, nodes[u].child + 1})
          if (!is_leaf(c)) q.emplace_back(c, d + 1);
      }
      for (auto [u, d] : exits) {
        (void)d;
        if (win_of_root[u] < 0) {
          win_of_root[u] = (int32_t)members.size();
          members.emplace_back();
          ldepth.emplace_back();
          roots.push_back(u);
        }
      }
      members[w] = std::move(mem);
      ldepth[w] = std::move(dep);
    }
    const uint32_t nw = (uint32_t)members.size();
    std::vector<uint32_t> base(nw);
    uint64_t total = 0;
    for (uint32_t w = 0; w < nw; ++w) {
      base[w] = (uint32_t)total;
      total += members[w].size();
    }
    if (16 * (total + 32) >= (1u << 30)) fail(ST_ERR_ARGUMENT, "tree too large for speculative windows");
    wt.entries.resize(total + 32, SEntry{0.0f, 0u, 0u, 0u});
    std::vector<int32_t> lane_of(n, -1);
    for (uint32_t w = 0; w < nw; ++w) {
      const auto& mem = members[w];
      uint32_t h = 0;
      for (uint32_t j = 0; j < mem.size(); ++j) {
        lane_of[mem[j]] = (int32_t)j;
        h = std::max(h, ldepth[w][j] + 1);
      }
      const uint32_t steps = ceil_log2(h);
      wt.max_steps = std::max(wt.max_steps, steps);
      auto code = [&](uint32_t c) -> uint32_t {
        if (is_leaf(c)) return kLeafBit | leaf_code[c];
        if (lane_of[c] >= 0) return (uint32_t)lane_of[c];
        return kExitBit | (16u * base[win_of_root[c]]);  // byte offset of the window
      };
      for (uint32_t j = 0; j < mem.size(); ++j) {
        const st_node& nd = nodes[mem[j]];
        SEntry e;
        e.thr = nd.threshold;
        e.attr_steps = (4u * nd.attribute) | (steps << 24);
        e.left = code(nd.child);
        e.right = code(nd.child + 1);
        wt.entries[base[w] + j] = e;
      }
      for (uint32_t j = 0; j < mem.size(); ++j) lane_of[mem[j]] = -1;
    }
    wt.root_code = kExitBit | 0u;
    wt.windows = nw;
    return wt;
  }

  Dev& device(int d) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = dev.find(d);
    if (it != dev.end()) return it->second;
    Dev dv;
    CK(cudaMalloc(&dv.wide, nodes.size() * sizeof(st_node)));
    CK(cudaMemcpy(dv.wide, nodes.data(), nodes.size() * sizeof(st_node), cudaMemcpyHostToDevice));
    if (compact_ok) {
      const size_t bytes = ((compact.size() * sizeof(CNode) + 15) & ~size_t(15)) + 16;
      CK(cudaMalloc(&dv.compact, bytes));
      CK(cudaMemset(dv.compact, 0, bytes));
      CK(cudaMemcpy(dv.compact, compact.data(), compact.size() * sizeof(CNode),
                    cudaMemcpyHostToDevice));
    }
    {
      std::vector<uint32_t> map;
      for (uint32_t i = 0; i < nodes.size(); ++i)
        if (!is_leaf(i)) map.push_back(i);
      map.push_back(0);  // keep the allocation non-empty
      CK(cudaMalloc(&dv.internal_map, map.size() * 4));
      CK(cudaMemcpy(dv.internal_map, map.data(), map.size() * 4, cudaMemcpyHostToDevice));
    }
    if (leaf_table) {
      CK(cudaMalloc(&dv.leaf_tbl, leaf_classes.size() * 4));
      CK(cudaMemcpy(dv.leaf_tbl, leaf_classes.data(), leaf_classes.size() * 4,
                    cudaMemcpyHostToDevice));
    }
    return dev.emplace(d, dv).first->second;
  }

  SEntry* device_windows(int d, uint32_t G, uint32_t H, const WinTable& wt) {
    Dev& dv = device(d);
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(G, H);
    auto it = dv.wins.find(key);
    if (it != dv.wins.end()) return it->second;
    SEntry* p = nullptr;
    CK(cudaMalloc(&p, wt.entries.size() * sizeof(SEntry)));
    CK(cudaMemcpy(p, wt.entries.data(), wt.entries.size() * sizeof(SEntry), cudaMemcpyHostToDevice));
    dv.wins[key] = p;
    return p;
  }
};

struct st_forest {
  std::vector<CNode> compact;      // trees concatenated, each starting 16-byte aligned
  std::vector<uint32_t> offsets;   // first node of each tree (+ end sentinel)
  std::vector<uint32_t> tree_bytes;  // bytes per tree rounded up to 16 (bulk-copy size)
  uint32_t max_tree_bytes = 0;
  uint32_t t_count = 0, n_classes = 0, abits = 1, max_attribute = 0;
  std::mutex mu;
  struct Dev {
    CNode* nodes = nullptr;
    uint32_t* offsets = nullptr;
    uint32_t* tree_bytes = nullptr;
  };
  std::map<int, Dev> dev;
  ~st_forest() {
    int cur = -1;
    cudaGetDevice(&cur);
    for (auto& kv : dev) {
      if (cudaSetDevice(kv.first) != cudaSuccess) continue;
      cudaFree(kv.second.nodes);
      cudaFree(kv.second.offsets);
      cudaFree(kv.second.tree_bytes);
    }
    if (cur >= 0) cudaSetDevice(cur);
  }
  Dev& device(int d) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = dev.find(d);
    if (it != dev.end()) return it->second;
    Dev dv;
    CK(cudaMalloc(&dv.nodes, compact.size() * sizeof(CNode) + 16));
    CK(cudaMemcpy(dv.nodes, compact.data(), compact.size() * sizeof(CNode), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dv.offsets, offsets.size() * 4));
    CK(cudaMemcpy(dv.offsets, offsets.data(), offsets.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dv.tree_bytes, tree_bytes.size() * 4));
    CK(cudaMemcpy(dv.tree_bytes, tree_bytes.data(), tree_bytes.size() * 4, cudaMemcpyHostToDevice));
    return dev.emplace(d, dv).first->second;
  }
};

namespace {

// ---------------------------------------------------------------------------
// Tree construction
// ---------------------------------------------------------------------------
void validate_links(const st_node* nodes, uint32_t n, const char* what) {
  if (n == 0) fail(ST_ERR_ARGUMENT, "encoded tree requires at least one node");
  for (uint32_t i = 0; i < n; ++i) {
    const st_node& nd = nodes[i];
    if (nd.class_id != ST_NO_CLASS) continue;
    if (nd.child + 1 >= n || nd.child + 1 < nd.child)
      fail(ST_ERR_ARGUMENT, std::string(what) + ": node " + std::to_string(i) + ": child index " +
                                std::to_string(nd.child) + " out of range");
    if (nd.child <= i)
      fail(ST_ERR_ARGUMENT, std::string(what) + ": node " + std::to_string(i) +
                                ": non-BFS child link: child " + std::to_string(nd.child) +
                                " does not point forward");
  }
}

uint32_t bits_for(uint64_t v) {  // bits to hold values 0..v
  uint32_t b = 1;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

// Compact meta for an internal node: (8*child) << abits | 4*attr.
bool compact_fits(uint32_t n, uint32_t max_attribute, uint32_t* abits) {
  *abits = bits_for(4ull * max_attribute);
  return *abits < 31 && ((8ull * n) << *abits) < (1ull << 31);
}

std::unique_ptr<st_tree> make_tree(const st_node* nodes, uint32_t n) {
  validate_links(nodes, n, "tree");
  auto t = std::make_unique<st_tree>();
  t->nodes.assign(nodes, nodes + n);
  st_tree_info& in = t->info;
  in.nodes = n;
  std::vector<uint32_t> depth(n, 0);
  for (uint32_t i = 0; i < n; ++i) {
    const st_node& nd = nodes[i];
    in.max_attribute = std::max(in.max_attribute, nd.attribute);  // tree.cpp:47: all nodes
    if (nd.class_id != ST_NO_CLASS) {
      ++in.leaves;
      in.depth = std::max(in.depth, depth[i]);
      in.max_class = std::max(in.max_class, nd.class_id);
      if (nd.class_id >= kLeafBit) t->leaf_table = true;
    } else {
      ++in.internal;
      depth[nd.child] = std::max(depth[nd.child], depth[i] + 1);
      depth[nd.child + 1] = std::max(depth[nd.child + 1], depth[i] + 1);
    }
  }
  t->leaf_code.assign(n, 0);
  for (uint32_t i = 0; i < n; ++i) {
    if (nodes[i].class_id == ST_NO_CLASS) continue;
    if (t->leaf_table) {
      t->leaf_code[i] = (uint32_t)t->leaf_classes.size();
      t->leaf_classes.push_back(nodes[i].class_id);
    } else {
      t->leaf_code[i] = nodes[i].class_id;
    }
  }
  t->compact_ok = compact_fits(n, in.max_attribute, &t->abits);
  if (t->compact_ok) {
    t->compact.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
      const st_node& nd = nodes[i];
      if (nd.class_id != ST_NO_CLASS)
        t->compact[i] = CNode{nd.threshold, kLeafBit | t->leaf_code[i]};
      else
        t->compact[i] = CNode{nd.threshold, ((8u * nd.child) << t->abits) | (4u * nd.attribute)};
    }
  }
  in.compact = t->compact_ok ? 1 : 0;
  return t;
}

// ---------------------------------------------------------------------------
// Launch helpers
// ---------------------------------------------------------------------------
int blocks_for(const void* fn, size_t smem, int dev, uint32_t blocks_per_sm, uint64_t n_tiles,
               uint32_t warps = kWarpsPerCta) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, bool> attr_set;
  static std::map<std::tuple<const void*, size_t, int, uint32_t>, int> occ_cache;
  const DevProps pr = dev_props(dev);
  if (smem > pr.smem_optin)
    fail(ST_ERR_ARGUMENT, "kernel needs " + std::to_string(smem) + " B of shared memory (max " +
                              std::to_string(pr.smem_optin) + ")");
  int occ = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    // The dynamic-smem ceiling is set once per (kernel, device) to the opt-in
    // maximum, so launches of any size after it stay valid.
    auto akey = std::make_pair(fn, dev);
    if (!attr_set.count(akey)) {
      CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pr.smem_optin));
      attr_set[akey] = true;
    }
    auto key = std::make_tuple(fn, smem, dev, warps);
    auto it = occ_cache.find(key);
    if (it != occ_cache.end()) {
      occ = it->second;
    } else {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, (int)warps * 32, smem));
      if (occ < 1) fail(ST_ERR_ARGUMENT, "kernel configuration does not fit on an SM");
      occ_cache[key] = occ;
    }
  }
  uint64_t blocks = (uint64_t)pr.sms * (blocks_per_sm ? std::min<uint32_t>(blocks_per_sm, occ) : occ);
  const uint64_t need = (n_tiles + warps - 1) / warps;
  return (int)std::max<uint64_t>(1, std::min(blocks, need));
}

// Clear a stale, non-sticky error left by an earlier runtime call (ours or the
// host application's) so the post-launch check reports this launch only.
void clear_stale_error() { (void)cudaGetLastError(); }

void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(ST_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  ++g_launches;
}

void check_common(uint64_t m, uint32_t a, uint64_t& ld, int layout, uint32_t max_attribute) {
  if (a == 0) fail(ST_ERR_ARGUMENT, "dataset arity must be >= 1");
  if (layout != ST_LAYOUT_AOS && layout != ST_LAYOUT_SOA) fail(ST_ERR_ARGUMENT, "unknown layout");
  if (ld == 0) ld = layout == ST_LAYOUT_AOS ? a : m;
  if (layout == ST_LAYOUT_AOS && ld < a) fail(ST_ERR_ARGUMENT, "AoS ld must be >= arity");
  if (layout == ST_LAYOUT_SOA && ld < m) fail(ST_ERR_ARGUMENT, "SoA ld must be >= record count");
  if (ld > 0xFFFFFFFFull) fail(ST_ERR_ARGUMENT, "ld too large");
  // check_attribute_range (eval_serial.cpp:10-17), before any work
  if (max_attribute >= a)
    fail(ST_ERR_ARGUMENT, "tree reads attribute " + std::to_string(max_attribute) +
                              " but records have arity " + std::to_string(a));
}

// ---- TMA tensor maps ---------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (EncodeTiledFn) nullptr;
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// Record staging plan for one launch.
struct Staging {
  int loader = kScalar;
  uint32_t S = 1;           // records per lane per tile (tile = 32*S records)
  uint32_t ns = 1;          // pipeline stages per warp
  uint32_t stage_bytes = 0;
  uint32_t warps = kWarpsPerCta;  // CTA width
  CUtensorMap tmap{};
  size_t tile_smem() const {  // all warps' stages + their mbarriers
    return loader == kDirect ? 0 : (size_t)warps * ns * (stage_bytes + 8u);
  }
};

uint32_t round1024(uint64_t b) { return (uint32_t)((b + 1023) & ~uint64_t(1023)); }

// TMA applies to packed AoS, 16 B-aligned, with a tile of <= 256 rows of 32 floats.
bool tma_ok(const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout, uint32_t S) {
  if (layout != ST_LAYOUT_AOS || ld != a) return false;
  if ((reinterpret_cast<uintptr_t>(x) & 15u) != 0) return false;
  if (32ull * S * a > 8192) return false;         // box rows = 32*S*a/32 <= 256
  if (m < 32ull * S) return false;                 // no full tile: nothing for TMA to move
  if (m * (uint64_t)a / 32 >= (1ull << 31)) return false;
  return encode_tiled() != nullptr;
}

void make_tmap(Staging& st, const float* x, uint64_t m, uint32_t a) {
  const cuuint64_t dims[2] = {32, (cuuint64_t)(m * (uint64_t)a / 32)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {32, 32u * st.S * a / 32u};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_tiled()(&st.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x),
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
}

// Choose loader, S and stages.  `fixed` = shared bytes needed besides the
// record stages (tree / windows / counters).
Staging plan_staging(const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout, uint32_t S,
                     uint32_t want_ns, size_t fixed, const DevProps& pr) {
  Staging st;
  st.S = S;
  const bool tma = tma_ok(x, m, a, ld, layout, S);
  st.loader = tma ? kTma : (layout == ST_LAYOUT_SOA ? kSoa : kScalar);
  st.stage_bytes = round1024(32ull * S * a * 4);
  if (tma) {
    // ~100 KB per CTA so two CTAs (16 warps) share an SM: 2-4 stages per warp
    // Two stages per warp (one tile walked, one in flight) measured best on
    // C2: more bytes in flight per SM did not raise HBM throughput.
    const uint32_t ns = want_ns ? want_ns : 2;
    st.ns = std::max<uint32_t>(1, std::min<uint32_t>(ns, 8));
    while (st.ns > 1 && fixed + 1024 + st.tile_smem() > pr.smem_optin) --st.ns;
    make_tmap(st, x, m, a);
  } else {
    st.ns = 1;
  }
  if (fixed + 1024 + st.tile_smem() > pr.smem_optin) {
    st.loader = kDirect;  // records too wide to stage: read features from global
    st.S = 1;
    st.ns = 1;
  }
  return st;
}

uint32_t pick_warps(uint32_t want, const Staging& st, size_t fixed, const DevProps& pr) {
  auto fits = [&](uint32_t w) {
    return fixed + 1024 + (st.loader == kDirect ? 0 : (size_t)w * st.ns * (st.stage_bytes + 8u)) +
               (size_t)w * 3 * 128 <= pr.smem_optin;
  };
  if (want) {
    const uint32_t w = std::max<uint32_t>(1, std::min<uint32_t>(want, 32));
    if (!fits(w)) fail(ST_ERR_ARGUMENT, "warps_per_cta " + std::to_string(w) + " does not fit in shared memory");
    return w;
  }
  if (st.loader == kTma) {
    // ~128 KB of record stages in flight per SM saturated HBM in every sweep
    // (C2: 16 warps x 2 x 4 KB; C5: 32 warps x 2 x 2 KB); use one wide CTA so
    // a shared-memory tree is staged once per SM.
    uint32_t w = (uint32_t)std::min<size_t>(32, std::max<size_t>(8, (128u << 10) / ((size_t)st.ns * st.stage_bytes)));
    while (w > 8 && !fits(w)) w -= 8;
    if (fits(w)) return w;
  }
  if (fixed > 16 * 1024)
    for (uint32_t w : {32u, 16u})
      if (fits(w)) return w;
  return kWarpsPerCta;
}

// Persistent-grid width: on large TMA-streamed inputs 2 CTAs (16 warps) per SM
// saturate HBM and beat the occupancy maximum (C2 sweep, profiles/); small
// inputs use every resident CTA to hide latency.
uint32_t default_bps(uint32_t want, const Staging& st, uint64_t m, const DevProps& pr) {
  if (want) return want;
  if (st.loader != kTma) return 0;
  // one wide CTA per SM carries the ~128 KB of stages (pick_warps); more CTAs
  // only pay on inputs too small to fill the SMs
  const uint64_t tiles = m / (32ull * st.S);
  return tiles >= (uint64_t)pr.sms * st.warps * 16 ? std::max<uint32_t>(1, 16 / st.warps) : 0u;
}

PipeArgs pipe_args(const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout) {
  PipeArgs p{};
  p.x = x;
  p.m = m;
  p.a = a;
  p.ld = (uint32_t)ld;
  p.layout_soa = layout == ST_LAYOUT_SOA ? 1u : 0u;
  return p;
}

// ---- data kernel dispatch ------------------------------------------------
template <int A, int S, int TLOC, int LOADER, int CAP>
void launch_data_t(const DataArgs& d, const Staging& stg, const ConstTree<CAP>* ct, size_t smem,
                   int dev, uint32_t bps, cudaStream_t s) {
  auto fn = k_data<A, S, TLOC, LOADER, CAP>;
  const uint64_t n_tiles = (d.p.m + 32 * S - 1) / (32 * S);
  const int blocks = blocks_for((const void*)fn, smem, dev, bps, n_tiles, stg.warps);
  static const ConstTree<1> dummy{};
  clear_stale_error();
  if constexpr (CAP == 1) {
    fn<<<blocks, stg.warps * 32, smem, s>>>(d, stg.tmap, ct ? *ct : dummy);
  } else {
    fn<<<blocks, stg.warps * 32, smem, s>>>(d, stg.tmap, *ct);
  }
  check_launch();
}

template <int A, int S, int LOADER>
void launch_data_tloc(int tloc, const DataArgs& d, const Staging& stg, const st_tree* t,
                      size_t smem, int dev, uint32_t bps, cudaStream_t s) {
  switch (tloc) {
    case ST_TREE_SHARED:
      if constexpr ((A == 8 || A == 16) && LOADER == kTma) {
        if (d.record_regs) return launch_data_t<A, S, kSharedReg, LOADER, 1>(d, stg, nullptr, smem, dev, bps, s);
      }
      return launch_data_t<A, S, kShared, LOADER, 1>(d, stg, nullptr, smem, dev, bps, s);
    case ST_TREE_GLOBAL:
      return launch_data_t<A, S, kGlobal, LOADER, 1>(d, stg, nullptr, smem, dev, bps, s);
    case ST_TREE_CONSTANT: {
      if constexpr (LOADER == kTma) {
        if (t->compact.size() <= 512) {
          ConstTree<512> ct{};
          std::copy(t->compact.begin(), t->compact.end(), ct.n);
          return launch_data_t<A, S, kConst, LOADER, 512>(d, stg, &ct, smem, dev, bps, s);
        }
        auto ct = std::make_unique<ConstTree<4000>>();
        std::copy(t->compact.begin(), t->compact.end(), ct->n);
        return launch_data_t<A, S, kConst, LOADER, 4000>(d, stg, ct.get(), smem, dev, bps, s);
      }
      break;
    }
    default:
      break;
  }
  return launch_data_t<A, S, kWide, LOADER, 1>(d, stg, nullptr, smem, dev, bps, s);
}

// Compile-time arities with a TMA fast path; everything else runs A = 0.
bool ct_arity(uint32_t a) { return a == 8 || a == 16 || a == 32 || a == 64; }

uint32_t choose_S(uint32_t a, uint32_t want) {
  // instantiated: a=8 {1,2,4}, a=16 {1,2,4}, a=32 {1,2}, others {1}
  const uint32_t maxS = (a == 8 || a == 16) ? 4 : a == 32 ? 2 : 1;
  // predicated walk (k_data data_step): independent chains per lane pay off
  // where a tile is small -- C3 (a = 8): S = 4 0.63 ms vs S = 2 0.67 ms for 32
  // frames; C2 (a = 32): S = 2 0.307 vs S = 1 0.321 ms (profiles/r1_sweep_*)
  if (want == 0) want = a <= 8 ? 4 : a == 32 ? 2 : 1;
  uint32_t S = 1;
  while (S * 2 <= std::min(want, maxS)) S *= 2;
  return S;
}

template <int A>
void launch_data_a(const Staging& stg, int tloc, const DataArgs& d, const st_tree* t, size_t smem,
                   int dev, uint32_t bps, cudaStream_t s) {
  if constexpr (A == 8 || A == 16) {
    if (stg.S == 4) return launch_data_tloc<A, 4, kTma>(tloc, d, stg, t, smem, dev, bps, s);
  }
  if constexpr (A == 8 || A == 16 || A == 32) {
    if (stg.S == 2) return launch_data_tloc<A, 2, kTma>(tloc, d, stg, t, smem, dev, bps, s);
  }
  return launch_data_tloc<A, 1, kTma>(tloc, d, stg, t, smem, dev, bps, s);
}

void eval_data_device(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                      const st_geom& g, uint32_t* labels, cudaStream_t s, int dev) {
  st_tree::Dev& dv = t->device(dev);
  const DevProps pr = dev_props(dev);
  DataArgs d{};
  d.p = pipe_args(x, m, a, ld, layout);
  d.nodes = dv.compact;
  d.wide = dv.wide;
  d.n_nodes = (uint32_t)t->nodes.size();
  d.abits = t->abits;
  d.leaf_class = dv.leaf_tbl;
  d.labels = labels;
  // records walked from registers: default for 8-attribute records; 16 on request
  d.record_regs = (g.record_regs == 1 || (g.record_regs == 0 && a == 8)) ? 1u : 0u;

  const uint32_t tree_bytes = round1024(t->nodes.size() * sizeof(CNode));
  int tloc = g.tree_loc;
  if (!t->compact_ok) tloc = kWide;
  else if (tloc == ST_TREE_AUTO) tloc = tree_bytes <= 96 * 1024 ? ST_TREE_SHARED : ST_TREE_GLOBAL;
  if (tloc == ST_TREE_CONSTANT && t->compact.size() > 4000) tloc = ST_TREE_GLOBAL;
  const uint32_t S0 = ct_arity(a) ? choose_S(a, g.samples_per_thread) : 1;
  // Records walked from registers release their tile before the walk, so one
  // stage per warp already double-buffers (next TMA in flight during the
  // walk) and the saved shared memory buys twice the warps (C3 x 32 frames:
  // 0.566 vs 0.615 ms, profiles/r1_sweep_C3x32_regs1.json).
  const uint32_t want_ns = g.stages ? g.stages : (d.record_regs && tloc == ST_TREE_SHARED ? 1u : 0u);
  Staging stg = plan_staging(x, m, a, ld, layout, S0, want_ns,
                             tloc == ST_TREE_SHARED ? tree_bytes : 0, pr);
  if (tloc == ST_TREE_SHARED && tree_bytes + 1024 + stg.tile_smem() > pr.smem_optin) {
    tloc = ST_TREE_GLOBAL;
    stg = plan_staging(x, m, a, ld, layout, S0, g.stages, 0, pr);
  }
  if (tloc == ST_TREE_CONSTANT && stg.loader != kTma) tloc = ST_TREE_GLOBAL;
  // A large shared-memory tree is staged once per CTA: widen the CTA so that
  // one copy serves up to 32 warps instead of capping the SM at one 8-warp CTA.
  stg.warps = pick_warps(g.warps_per_cta, stg, tloc == ST_TREE_SHARED ? tree_bytes : 0, pr);
  uint32_t want_bps = g.blocks_per_sm;
  // Small inputs (< 8 tiles per warp at 32 warps/SM, e.g. C1's 1M records)
  // are ramp-up bound: four 8-warp CTAs per SM stage their tree copies
  // faster than one 32-warp CTA (C1: 17.0 vs 19.3 us, profiles/r1_sweep_C1x1_small_flush.json).
  const uint64_t tiles_total = m / (32ull * stg.S);
  if (!g.warps_per_cta && !g.blocks_per_sm && stg.loader == kTma && tloc == ST_TREE_SHARED &&
      tiles_total < (uint64_t)pr.sms * 32 * 8 &&
      4 * (1024 + tree_bytes + (size_t)kWarpsPerCta * stg.ns * (stg.stage_bytes + 8u)) <= pr.smem_per_sm) {
    stg.warps = kWarpsPerCta;
    want_bps = 4;
  }
  d.ns = stg.ns;
  d.stage_bytes = stg.stage_bytes;
  d.tree_bytes = tloc == ST_TREE_SHARED ? tree_bytes : 0;
  const size_t smem = 1024 + d.tree_bytes + stg.tile_smem();
  const uint32_t bps = default_bps(want_bps, stg, m, pr);
  if (stg.loader == kTma && ct_arity(a)) {
    switch (a) {
      case 8: return launch_data_a<8>(stg, tloc, d, t, smem, dev, bps, s);
      case 16: return launch_data_a<16>(stg, tloc, d, t, smem, dev, bps, s);
      case 32: return launch_data_a<32>(stg, tloc, d, t, smem, dev, bps, s);
      case 64: return launch_data_a<64>(stg, tloc, d, t, smem, dev, bps, s);
    }
  }
  switch (stg.loader) {
    case kTma: return launch_data_tloc<0, 1, kTma>(tloc, d, stg, t, smem, dev, bps, s);
    case kDirect:
      return launch_data_tloc<0, 1, kDirect>(tloc == ST_TREE_CONSTANT ? ST_TREE_GLOBAL : tloc, d,
                                             stg, t, smem, dev, bps, s);
    default:
      return launch_data_tloc<0, 1, kScalar>(tloc == ST_TREE_CONSTANT ? ST_TREE_GLOBAL : tloc, d,
                                             stg, t, smem, dev, bps, s);
  }
}

uint32_t env_u32(const char* name, uint32_t dflt);

// ---- speculative kernel dispatch -----------------------------------------
template <int A, int LOADER, bool WS, bool EXACT, int STEPS>
void launch_spec_k(const SpecArgs& sa, const Staging& stg, size_t smem, int dev, uint32_t bps,
                   cudaStream_t s) {
  auto fn = k_spec<A, LOADER, WS, EXACT, STEPS>;
  const uint64_t n_tiles = (sa.p.m + 31) / 32;
  const int blocks = blocks_for((const void*)fn, smem, dev, bps, n_tiles, stg.warps);
  clear_stale_error();
  fn<<<blocks, stg.warps * 32, smem, s>>>(sa, stg.tmap);
  check_launch();
}

// Fast path: the doubling count is a compile-time constant for the usual
// window heights (steps 0..3); EXACT (reference counters) and taller windows
// use a runtime count.
template <int A, int LOADER, bool WS>
void launch_spec_steps(const SpecArgs& sa, const Staging& stg, size_t smem, int dev, uint32_t bps,
                       cudaStream_t s) {
  if (sa.iters) return launch_spec_k<A, LOADER, WS, true, -1>(sa, stg, smem, dev, bps, s);
  switch (sa.smax) {
    case 0: return launch_spec_k<A, LOADER, WS, false, 0>(sa, stg, smem, dev, bps, s);
    case 1: return launch_spec_k<A, LOADER, WS, false, 1>(sa, stg, smem, dev, bps, s);
    case 2: return launch_spec_k<A, LOADER, WS, false, 2>(sa, stg, smem, dev, bps, s);
    case 3: return launch_spec_k<A, LOADER, WS, false, 3>(sa, stg, smem, dev, bps, s);
    default: return launch_spec_k<A, LOADER, WS, false, -1>(sa, stg, smem, dev, bps, s);
  }
}

template <int A, bool WS, int STEPS, int SR>
void launch_spec_ring_k(const SpecRingArgs& ra, const Staging& stg, size_t smem, int dev,
                        uint32_t warps, cudaStream_t s) {
  auto fn = k_spec_ring<A, WS, STEPS, SR>;
  const uint64_t n_tiles = (ra.s.p.m + 31) / 32;
  const int blocks = blocks_for((const void*)fn, smem, dev, 0, n_tiles * warps, warps);
  clear_stale_error();
  fn<<<blocks, warps * 32, smem, s>>>(ra, stg.tmap);
  check_launch();
}

template <int A, bool WS, int STEPS>
void launch_spec_ring_sr(uint32_t sr, const SpecRingArgs& ra, const Staging& stg, size_t smem, int dev,
                         uint32_t warps, cudaStream_t s) {
  if (sr >= 2) return launch_spec_ring_k<A, WS, STEPS, 2>(ra, stg, smem, dev, warps, s);
  return launch_spec_ring_k<A, WS, STEPS, 1>(ra, stg, smem, dev, warps, s);
}

template <int A>
void launch_spec_ring(bool ws, uint32_t sr, const SpecRingArgs& ra, const Staging& stg, size_t smem,
                      int dev, uint32_t warps, cudaStream_t s) {
#define ST_RING(WSV, ST) return launch_spec_ring_sr<A, WSV, ST>(sr, ra, stg, smem, dev, warps, s)
  if (ws) {
    switch (ra.s.smax) {
      case 0: ST_RING(true, 0);
      case 1: ST_RING(true, 1);
      case 2: ST_RING(true, 2);
      case 3: ST_RING(true, 3);
      default: ST_RING(true, -1);
    }
  }
  switch (ra.s.smax) {
    case 0: ST_RING(false, 0);
    case 1: ST_RING(false, 1);
    case 2: ST_RING(false, 2);
    case 3: ST_RING(false, 3);
    default: ST_RING(false, -1);
  }
#undef ST_RING
}

template <int A, int LOADER>
void launch_spec_t(bool win_shared, const SpecArgs& sa, const Staging& stg, size_t smem, int dev,
                   uint32_t bps, cudaStream_t s) {
  if (win_shared) return launch_spec_steps<A, LOADER, true>(sa, stg, smem, dev, bps, s);
  return launch_spec_steps<A, LOADER, false>(sa, stg, smem, dev, bps, s);
}

void spec_geometry(const st_tree* t, const st_geom& g, uint32_t& G, uint32_t& H) {
  G = g.group_lanes;
  if (G == 0) {
    const uint32_t I = std::max<uint32_t>(1, t->info.internal);
    if (I <= 32) {
      // whole tree in one record group: the paper's Proc. 5 geometry
      // (15 internal nodes -> its half-warp of 16 lanes)
      G = 1;
      while (G < I) G *= 2;
    } else {
      // larger trees: 3-node windows in 4-lane groups (two levels per window,
      // one shfl doubling) measured fastest on C2 among genuine speculation
      G = 4;
    }
  }
  if (G > 32 || (G & (G - 1)) != 0)
    fail(ST_ERR_ARGUMENT, "group_lanes must be a power of two <= 32 on the GPU, got " +
                              std::to_string(g.group_lanes));
  H = g.window_levels;
  if (H == 0) {
    if (t->info.internal <= G) {
      // whole tree in one window: the paper's Proc. 5 geometry (mapped lanes)
      H = std::max<uint32_t>(1, t->info.depth);
    } else {
      // complete-level windows: largest H with 2^H - 1 <= G
      H = 1;
      while ((2u << H) - 1 <= G) ++H;
    }
  }
}

// Reference counters for trees with more than 32 internal nodes: CTA-scope
// whole-tree speculation (k_spec_exact_cta).
void eval_spec_exact_cta(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                         int layout, uint32_t k, uint32_t* labels, st_stats* stats, cudaStream_t s,
                         int dev) {
  st_tree::Dev& dv = t->device(dev);
  const DevProps pr = dev_props(dev);
  SpecExactArgs ea{};
  ea.p = pipe_args(x, m, a, ld, layout);
  ea.nodes = dv.wide;
  ea.map = dv.internal_map;
  ea.n = (uint32_t)t->nodes.size();
  ea.I = t->info.internal;
  ea.k = k ? k : 1;
  ea.labels = labels;
  ea.iters = stats->iterations;
  ea.steps = stats->doubling_steps;
  const size_t smem = 8ull * t->nodes.size() + 16;
  if (smem > pr.smem_optin) fail(ST_ERR_ARGUMENT, "tree too large for exact speculative counters");
  const uint32_t threads = std::min<uint32_t>(1024, std::max<uint32_t>(32, (ea.I + 31) / 32 * 32));
  auto fn = k_spec_exact_cta;
  static std::mutex mu;
  static std::map<int, bool> attr;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!attr.count(dev)) {
      CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)pr.smem_optin));
      attr[dev] = true;
    }
  }
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, (int)threads, smem));
  const uint64_t blocks = std::min<uint64_t>(m, (uint64_t)pr.sms * std::max(occ, 1));
  clear_stale_error();
  fn<<<(unsigned)blocks, threads, smem, s>>>(ea);
  check_launch();
}

void eval_spec_device(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                      const st_geom& g, uint32_t* labels, st_stats* stats, cudaStream_t s, int dev) {
  if (stats && t->info.internal > 32) {
    // counters are defined by whole-tree speculation (the reference law)
    return eval_spec_exact_cta(t, x, m, a, ld, layout, g.reductions, labels, stats, s, dev);
  }
  st_geom gg = g;
  if (stats) {
    // whole tree in one record group so the counters follow the reference law
    uint32_t G = 1;
    while (G < std::max<uint32_t>(1, t->info.internal)) G *= 2;
    gg.group_lanes = G;
    gg.window_levels = std::max<uint32_t>(1, t->info.depth);
  }
  uint32_t G, H;
  spec_geometry(t, gg, G, H);
  if (4ull * t->info.max_attribute >= (1u << 24))
    fail(ST_ERR_ARGUMENT, "speculative kernel requires attribute indices < 2^22");
  auto wt = t->windows(G, H);
  SEntry* wdev = t->device_windows(dev, G, H, *wt);
  st_tree::Dev& dv = t->device(dev);
  const DevProps pr = dev_props(dev);
  SpecArgs sa{};
  sa.p = pipe_args(x, m, a, ld, layout);
  sa.win = wdev;
  sa.n_entries = (uint32_t)wt->entries.size();
  sa.root_code = wt->root_code;
  sa.G = G;
  sa.smax = wt->max_steps;
  sa.k = g.reductions;
  sa.leaf_class = dv.leaf_tbl;
  sa.labels = labels;
  if (stats) {
    sa.iters = stats->iterations;
    sa.steps = stats->doubling_steps;
    if (!sa.iters || !sa.steps) fail(ST_ERR_ARGUMENT, "st_stats requires both arrays");
    if (sa.k == 0) sa.k = 1;  // counters follow the reference loop (k per root check)
  } else if (sa.k != 0) {
    // k without counters: same labels; the fixed-step path is used
    sa.k = 0;
  }
  const uint32_t win_bytes = round1024(wt->entries.size() * sizeof(SEntry));
  bool win_shared = win_bytes <= 96 * 1024;
  Staging stg = plan_staging(x, m, a, ld, layout, 1, g.stages, win_shared ? win_bytes : 0, pr);
  if (win_shared && win_bytes + 1024 + stg.tile_smem() > pr.smem_optin) {
    win_shared = false;
    stg = plan_staging(x, m, a, ld, layout, 1, g.stages, 0, pr);
  }
  sa.win_bytes = win_shared ? win_bytes : 0;
  if (stg.loader == kDirect) stg.ns = 1, stg.stage_bytes = 0;
  // speculative is issue/latency-bound: several 8-warp CTAs per SM (the
  // occupancy maximum) beat one wide CTA (C2: 0.52 vs 0.68 ms)
  stg.warps = g.warps_per_cta ? pick_warps(g.warps_per_cta, stg, sa.win_bytes, pr) : kWarpsPerCta;
  sa.ns = stg.ns;
  sa.stage_bytes = stg.stage_bytes;
  const size_t smem = 1024 + sa.win_bytes + (size_t)stg.warps * stg.ns * (stg.stage_bytes + 8u) +
                      (size_t)stg.warps * 3 * 128;  // + per-warp label/counter rows
  const uint32_t bps = g.blocks_per_sm;  // speculative is latency-bound: keep every resident CTA
  // CTA-shared ring (default for the fast path): up to 32 warps on one SM
  // share NS = warps + 12 tile slots; ~12 tiles in flight cover DRAM latency.
  if (stg.loader == kTma && !stats && g.pipeline != 1) {
    const size_t lb = 32 + 32 * 128;  // generation padding + ticket + per-warp label rows (<= 32 warps)
    const size_t budget = pr.smem_optin - 1024 - sa.win_bytes - lb;
    const size_t max_slots = budget / (stg.stage_bytes + 16u);
    const uint32_t warps = (uint32_t)std::min<size_t>(32, max_slots > 12 ? max_slots - 12 : 0);
    if (warps >= 4) {
      SpecRingArgs ra{};
      ra.s = sa;
      ra.n_slots = (uint32_t)std::min<size_t>(max_slots, warps + 12);
      // development / stress knob: any ring depth >= 1 must give exact labels
      if (const uint32_t ns = env_u32("ST_SPEC_RING_SLOTS", 0)) ra.n_slots = std::min<uint32_t>(ra.n_slots, ns);
      ra.unsafe_no_gen = env_u32("ST_SPEC_RING_UNSAFE_NO_GEN", 0);  // measurement of the handshake only
      const size_t rsmem = 1024 + sa.win_bytes + (size_t)ra.n_slots * (stg.stage_bytes + 8u) +
                           (((size_t)4 * ra.n_slots + 15) & ~size_t(15)) + 16 + (size_t)warps * 128;
      // record streams per group (samples_per_thread): one by default -- two
      // independent window chains per lane measured slower (C2 G = 4: 0.55 vs
      // 0.42 ms; profiles/r1_sweep_*_spec2.json)
      const uint32_t sr = g.samples_per_thread ? g.samples_per_thread : 1;
      switch (ct_arity(a) ? a : 0) {
        case 8: return launch_spec_ring<8>(win_shared, sr, ra, stg, rsmem, dev, warps, s);
        case 16: return launch_spec_ring<16>(win_shared, sr, ra, stg, rsmem, dev, warps, s);
        case 32: return launch_spec_ring<32>(win_shared, sr, ra, stg, rsmem, dev, warps, s);
        case 64: return launch_spec_ring<64>(win_shared, sr, ra, stg, rsmem, dev, warps, s);
        default: return launch_spec_ring<0>(win_shared, sr, ra, stg, rsmem, dev, warps, s);
      }
    }
  }
  if (stg.loader == kTma && ct_arity(a)) {
    switch (a) {
      case 8: return launch_spec_t<8, kTma>(win_shared, sa, stg, smem, dev, bps, s);
      case 16: return launch_spec_t<16, kTma>(win_shared, sa, stg, smem, dev, bps, s);
      case 32: return launch_spec_t<32, kTma>(win_shared, sa, stg, smem, dev, bps, s);
      case 64: return launch_spec_t<64, kTma>(win_shared, sa, stg, smem, dev, bps, s);
    }
  }
  switch (stg.loader) {
    case kTma: return launch_spec_t<0, kTma>(win_shared, sa, stg, smem, dev, bps, s);
    case kDirect: return launch_spec_t<0, kDirect>(win_shared, sa, stg, smem, dev, bps, s);
    default: return launch_spec_t<0, kScalar>(win_shared, sa, stg, smem, dev, bps, s);
  }
}

uint32_t resolve_algo(const st_tree* t, const st_geom& g, bool want_stats) {
  if (g.algo == ST_ALGO_DATA || g.algo == ST_ALGO_SPECULATIVE) return g.algo;
  if (g.algo != ST_ALGO_AUTO) fail(ST_ERR_ARGUMENT, "unknown algorithm " + std::to_string(g.algo));
  (void)t;
  return want_stats ? ST_ALGO_SPECULATIVE : ST_ALGO_DATA;
}

void eval_device_impl(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                      const st_geom* geom, uint32_t* labels, st_stats* stats, cudaStream_t s) {
  if (!t) fail(ST_ERR_ARGUMENT, "null tree");
  check_common(m, a, ld, layout, t->info.max_attribute);
  st_geom g{};
  if (geom) g = *geom;
  const uint32_t algo = resolve_algo(t, g, stats != nullptr);
  if (stats && algo != ST_ALGO_SPECULATIVE)
    fail(ST_ERR_ARGUMENT, "per-record stats are produced by the speculative kernel only");
  if (m == 0) return;  // empty dataset: empty output, no launch
  if (!x || !labels) fail(ST_ERR_ARGUMENT, "null data or label pointer");
  const int dev = current_device();
  if (algo == ST_ALGO_DATA)
    eval_data_device(t, x, m, a, ld, layout, g, labels, s, dev);
  else
    eval_spec_device(t, x, m, a, ld, layout, g, labels, stats, s, dev);
}

// ---- forest ----------------------------------------------------------------
template <int A, int LOADER>
void launch_forest_t(bool packed, const ForestArgs& fa, const Staging& stg, size_t smem, int dev,
                     cudaStream_t s) {
  const uint64_t n_tiles = (fa.p.m + 31) / 32;
  if (packed) {
    auto fn = k_forest<A, LOADER, true>;
    const int blocks = blocks_for((const void*)fn, smem, dev, 0, n_tiles, stg.warps);
    clear_stale_error();
    fn<<<blocks, stg.warps * 32, smem, s>>>(fa, stg.tmap);
  } else {
    auto fn = k_forest<A, LOADER, false>;
    const int blocks = blocks_for((const void*)fn, smem, dev, 0, n_tiles, stg.warps);
    clear_stale_error();
    fn<<<blocks, stg.warps * 32, smem, s>>>(fa, stg.tmap);
  }
  check_launch();
}

template <int A, int S, int U>
void launch_forest_smem(const Forest2Args& fa, const Staging& stg, size_t smem, int dev,
                        cudaStream_t s) {
  auto fn = k_forest_smem<A, S, U>;
  const uint64_t n_tiles = (fa.p.m + 32 * S - 1) / (32 * S);
  // warp 0 of each CTA is the tree producer: tiles are spread over warps - 1
  const int blocks = blocks_for((const void*)fn, smem, dev, 0,
                                n_tiles * stg.warps / std::max<uint32_t>(1, stg.warps - 1), stg.warps);
  clear_stale_error();
  fn<<<blocks, stg.warps * 32, smem, s>>>(fa, stg.tmap);
  check_launch();
}

template <int A, int S>
void launch_forest_u(uint32_t U, const Forest2Args& fa, const Staging& stg, size_t smem, int dev,
                     cudaStream_t s) {
  if constexpr (S == 1 && A > 0 && A <= 64) {  // the transposed-tile walk takes U chains
    if (U >= 4) return launch_forest_smem<A, S, 4>(fa, stg, smem, dev, s);
    if (U == 2) return launch_forest_smem<A, S, 2>(fa, stg, smem, dev, s);
  }
  return launch_forest_smem<A, S, 1>(fa, stg, smem, dev, s);
}

uint32_t env_u32(const char* name, uint32_t dflt) {  // development knobs for sweeps
  const char* v = std::getenv(name);
  return v && *v ? (uint32_t)std::strtoul(v, nullptr, 10) : dflt;
}

// Trees streamed through shared memory (packed votes, TMA-staged records).
bool forest_smem_path(st_forest* f, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                      int layout, uint32_t* labels, cudaStream_t s, int dev, const DevProps& pr) {
  if (!(f->n_classes <= 8 && f->t_count <= 255) || f->max_tree_bytes > 48 * 1024) return false;
  // one record per lane (the tile is transposed to attribute-major once per
  // round, which needs the record in registers); parallelism from wide CTAs
  const uint32_t S = 1;
  if (!tma_ok(x, m, a, ld, layout, S)) return false;
  Staging stg;
  stg.loader = kTma;
  stg.S = S;
  stg.ns = 1;
  stg.stage_bytes = round1024(32ull * S * a * 4);
  // Geometry: U trees walked per lane at once (U dependent-load chains), a
  // ring of NT tree slots, and as many consumer warps as the rest of shared
  // memory holds record tiles for.  The C4 sweep (profiles/r1_forest_sweep.json)
  // put U = 2 with NT = U + 2 first (8.3 ms vs 10.3 ms for U = 1, NT = 2):
  // the walk is bound by shared-memory wavefronts of the node loads, so more
  // chains than that only add ring slots at the expense of record tiles.
  const bool transposed = S == 1 && a <= 64 && ct_arity(a);
  const uint32_t U = std::max<uint32_t>(1, std::min<uint32_t>(4, env_u32("ST_FOREST_U", transposed ? 2 : 1)));
  uint32_t nt = env_u32("ST_FOREST_NT", 0);
  if (nt == 0) nt = U + 2;
  if (!transposed && U != 1) return false;
  stg.warps = 0;
  size_t fixed = 0;
  for (uint32_t n = nt; n >= std::max<uint32_t>(2, U) && !stg.warps; --n) {
    const size_t region = round1024((uint64_t)n * f->max_tree_bytes);
    const size_t base = 1024 + region + 16u * n;
    if (base >= pr.smem_optin) continue;
    uint32_t w = (uint32_t)std::min<size_t>(32, 1 + (pr.smem_optin - base) / (stg.stage_bytes + 8u));
    if (const uint32_t ww = env_u32("ST_FOREST_W", 0)) w = std::min(w, ww);
    if (w < 2) continue;
    stg.warps = w;
    nt = n;
    fixed = base;
  }
  if (!stg.warps) return false;
  make_tmap(stg, x, m, a);
  st_forest::Dev& dv = f->device(dev);
  Forest2Args fa{};
  fa.p = pipe_args(x, m, a, ld, layout);
  fa.nodes = dv.nodes;
  fa.offsets = dv.offsets;
  fa.t_count = f->t_count;
  fa.n_classes = f->n_classes;
  fa.abits = f->abits;
  fa.labels = labels;
  fa.stage_bytes = stg.stage_bytes;
  fa.tree_buf_bytes = f->max_tree_bytes;
  fa.n_tree_bufs = nt;
  fa.tree_region = round1024((uint64_t)nt * f->max_tree_bytes);
  fa.tree_bytes = dv.tree_bytes;
  const size_t smem = fixed + (size_t)(stg.warps - 1) * (stg.stage_bytes + 8u);
  switch (a) {
    case 8: return launch_forest_u<8, 1>(U, fa, stg, smem, dev, s), true;
    case 16: return launch_forest_u<16, 1>(U, fa, stg, smem, dev, s), true;
    case 32: return launch_forest_u<32, 1>(U, fa, stg, smem, dev, s), true;
    case 64: return launch_forest_u<64, 1>(U, fa, stg, smem, dev, s), true;
    default: return launch_forest_u<0, 1>(U, fa, stg, smem, dev, s), true;
  }
}

void forest_device_impl(st_forest* f, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                        int layout, uint32_t* labels, cudaStream_t s) {
  if (!f) fail(ST_ERR_ARGUMENT, "null forest");
  check_common(m, a, ld, layout, f->max_attribute);
  if (m == 0) return;
  if (!x || !labels) fail(ST_ERR_ARGUMENT, "null data or label pointer");
  const int dev = current_device();
  const DevProps pr = dev_props(dev);
  if (forest_smem_path(f, x, m, a, ld, layout, labels, s, dev, pr)) return;
  st_forest::Dev& dv = f->device(dev);
  ForestArgs fa{};
  fa.p = pipe_args(x, m, a, ld, layout);
  fa.nodes = dv.nodes;
  fa.offsets = dv.offsets;
  fa.t_count = f->t_count;
  fa.n_classes = f->n_classes;
  fa.abits = f->abits;
  fa.labels = labels;
  const bool packed = f->n_classes <= 8 && f->t_count <= 255;
  const size_t cnt_bytes = packed ? 0 : (size_t)kWarpsPerCta * 32 * f->n_classes * 4;  // 8-warp CTAs
  Staging stg = plan_staging(x, m, a, ld, layout, 1, 0, cnt_bytes, pr);
  fa.ns = stg.ns;
  fa.stage_bytes = stg.stage_bytes;
  const size_t smem = 1024 + stg.tile_smem() + cnt_bytes;
  if (stg.loader == kTma && ct_arity(a)) {
    switch (a) {
      case 8: return launch_forest_t<8, kTma>(packed, fa, stg, smem, dev, s);
      case 16: return launch_forest_t<16, kTma>(packed, fa, stg, smem, dev, s);
      case 32: return launch_forest_t<32, kTma>(packed, fa, stg, smem, dev, s);
      case 64: return launch_forest_t<64, kTma>(packed, fa, stg, smem, dev, s);
    }
  }
  switch (stg.loader) {
    case kTma: return launch_forest_t<0, kTma>(packed, fa, stg, smem, dev, s);
    case kDirect: return launch_forest_t<0, kDirect>(packed, fa, stg, smem, dev, s);
    default: return launch_forest_t<0, kScalar>(packed, fa, stg, smem, dev, s);
  }
}

// ---- host-buffer path --------------------------------------------------------
bool is_pinned_or_device(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice ||
         at.type == cudaMemoryTypeManaged;
}

// Per-device staging slots reused across host-path calls (a slot = stream +
// device record/label buffers + pinned label staging), so the H2D/kernel/D2H
// pipeline does not pay cudaMalloc/cudaFree per call.
struct Slot {
  cudaStream_t stream = nullptr;
  float* x = nullptr;
  size_t x_cap = 0;
  uint32_t* out[3] = {nullptr, nullptr, nullptr};  // labels + up to 2 counters
  uint32_t* pinned[3] = {nullptr, nullptr, nullptr};
  size_t out_cap = 0;
  bool busy = false;
};

class SlotPool {
 public:
  std::vector<Slot*> acquire(int dev, int n, size_t x_bytes, size_t rows) {
    std::lock_guard<std::mutex> lk(mu_);
    auto& v = pools_[dev];
    std::vector<Slot*> got;
    for (auto& sp : v)
      if (!sp->busy && (int)got.size() < n) got.push_back(sp.get());
    while ((int)got.size() < n) {
      v.push_back(std::make_unique<Slot>());
      got.push_back(v.back().get());
    }
    for (Slot* sl : got) {
      sl->busy = true;
      try {
        if (!sl->stream) CK(cudaStreamCreateWithFlags(&sl->stream, cudaStreamNonBlocking));
        if (sl->x_cap < x_bytes) {
          cudaFree(sl->x);
          sl->x = nullptr;
          sl->x_cap = 0;
          CK(cudaMalloc(&sl->x, x_bytes));
          sl->x_cap = x_bytes;
        }
        if (sl->out_cap < rows) {
          for (int k = 0; k < 3; ++k) {
            cudaFree(sl->out[k]);
            cudaFreeHost(sl->pinned[k]);
            sl->out[k] = nullptr;
            sl->pinned[k] = nullptr;
          }
          sl->out_cap = 0;
          for (int k = 0; k < 3; ++k) {
            CK(cudaMalloc(&sl->out[k], rows * 4));
            CK(cudaMallocHost(&sl->pinned[k], rows * 4));
          }
          sl->out_cap = rows;
        }
      } catch (...) {
        for (Slot* q : got) q->busy = false;
        throw;
      }
    }
    return got;
  }
  void release(const std::vector<Slot*>& s) {
    std::lock_guard<std::mutex> lk(mu_);
    for (Slot* sl : s) sl->busy = false;
  }

 private:
  std::mutex mu_;
  std::map<int, std::vector<std::unique_ptr<Slot>>> pools_;
};

SlotPool& slot_pool() {
  static SlotPool* p = new SlotPool();  // intentionally leaked: outlives static destructors
  return *p;
}

// Runs `kernel(x_dev, rows, ld_dev, labels_dev, extra_dev, stream)` over
// chunks of the host records with H2D / kernel / D2H overlapped across
// several streams.  Labels (and counters) come back through pinned staging
// when the caller's buffers are pageable.
template <class K>
void host_pipeline(const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                   uint32_t* labels, std::vector<std::pair<uint32_t*, uint32_t*>> extra_out,
                   K&& kernel) {
  constexpr int kStreams = 3;
  const uint64_t row_bytes = (uint64_t)a * 4;
  uint64_t chunk = std::max<uint64_t>(256, (64ull << 20) / row_bytes);  // ~64 MB of records
  chunk = (chunk + 255) / 256 * 256;
  chunk = std::min<uint64_t>(chunk, m);
  const uint64_t n_chunks = (m + chunk - 1) / chunk;
  const int ns = (int)std::min<uint64_t>(kStreams, n_chunks);
  const int dev = current_device();
  std::vector<Slot*> slots = slot_pool().acquire(dev, ns, chunk * row_bytes, chunk);
  struct Release {
    std::vector<Slot*>& s;
    ~Release() {
      for (Slot* sl : s) cudaStreamSynchronize(sl->stream);
      slot_pool().release(s);
    }
  } release{slots};
  const bool pinned_labels = is_pinned_or_device(labels);
  std::vector<uint32_t*> outs{labels};
  for (auto& e : extra_out) outs.push_back(e.first);
  // pending host copies out of pinned staging, per slot
  std::vector<std::pair<uint64_t, uint64_t>> pending(ns, {0, 0});
  auto drain = [&](int i) {
    if (pinned_labels || pending[i].second == 0) return;
    CK(cudaStreamSynchronize(slots[i]->stream));
    for (size_t k = 0; k < outs.size(); ++k)
      std::memcpy(outs[k] + pending[i].first, slots[i]->pinned[k], pending[i].second * 4);
    pending[i] = {0, 0};
  };
  for (uint64_t c = 0; c < n_chunks; ++c) {
    const int i = (int)(c % ns);
    Slot* sl = slots[i];
    drain(i);
    const uint64_t r0 = c * chunk;
    const uint64_t rows = std::min(chunk, m - r0);
    if (layout == ST_LAYOUT_AOS) {
      if (ld == a)
        CK(cudaMemcpyAsync(sl->x, x + r0 * a, rows * row_bytes, cudaMemcpyDefault, sl->stream));
      else
        CK(cudaMemcpy2DAsync(sl->x, row_bytes, x + r0 * ld, ld * 4, row_bytes, rows,
                             cudaMemcpyDefault, sl->stream));
    } else {
      CK(cudaMemcpy2DAsync(sl->x, rows * 4, x + r0, ld * 4, rows * 4, a, cudaMemcpyDefault,
                           sl->stream));
    }
    std::vector<uint32_t*> ex(sl->out + 1, sl->out + 1 + extra_out.size());
    kernel(sl->x, rows, layout == ST_LAYOUT_AOS ? (uint64_t)a : rows, sl->out[0], ex, sl->stream);
    for (size_t k = 0; k < outs.size(); ++k) {
      uint32_t* dst = pinned_labels ? outs[k] + r0 : sl->pinned[k];
      CK(cudaMemcpyAsync(dst, sl->out[k], rows * 4, cudaMemcpyDefault, sl->stream));
    }
    if (!pinned_labels) pending[i] = {r0, rows};
  }
  for (int i = 0; i < ns; ++i) {
    CK(cudaStreamSynchronize(slots[i]->stream));
    drain(i);
  }
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* st_last_error(void) { return g_error.c_str(); }
const char* st_version(void) { return "spectree_b200 0.1 (sm_100a)"; }
uint32_t st_last_launch_count(void) { return g_launches; }

void st_geom_default(st_geom* g) {
  if (g) std::memset(g, 0, sizeof(*g));
}

int st_device_count(int* count) {
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    *count = n;
  });
}

int st_tree_create(const st_node* nodes, uint32_t n, st_tree** out) {
  return guarded([&] {
    if (!out) fail(ST_ERR_ARGUMENT, "null output handle");
    if (!nodes && n) fail(ST_ERR_ARGUMENT, "null node array");
    *out = make_tree(nodes, n).release();
  });
}

void st_tree_destroy(st_tree* tree) { delete tree; }

int st_tree_get_info(const st_tree* tree, st_tree_info* out) {
  return guarded([&] {
    if (!tree || !out) fail(ST_ERR_ARGUMENT, "null argument");
    *out = tree->info;
    st_geom g{};
    uint32_t G, H;
    st_tree* t = const_cast<st_tree*>(tree);
    spec_geometry(t, g, G, H);
    out->spec_group_lanes = G;
    out->spec_windows = t->windows(G, H)->windows;
  });
}

int st_forest_create(const st_node* const* trees, const uint32_t* sizes, uint32_t t,
                     uint32_t n_classes, st_forest** out) {
  return guarded([&] {
    if (!out || (!trees && t) || (!sizes && t)) fail(ST_ERR_ARGUMENT, "null argument");
    if (t == 0) fail(ST_ERR_ARGUMENT, "forest requires at least one tree");
    if (n_classes == 0 || n_classes > 64) fail(ST_ERR_ARGUMENT, "forest n_classes must be in [1, 64]");
    auto f = std::make_unique<st_forest>();
    f->t_count = t;
    f->n_classes = n_classes;
    uint32_t maxattr = 0;
    uint64_t total = 0;
    for (uint32_t k = 0; k < t; ++k) {
      validate_links(trees[k], sizes[k], ("forest tree " + std::to_string(k)).c_str());
      for (uint32_t i = 0; i < sizes[k]; ++i) {
        maxattr = std::max(maxattr, trees[k][i].attribute);
        const uint32_t c = trees[k][i].class_id;
        if (c != ST_NO_CLASS && c >= n_classes)
          fail(ST_ERR_ARGUMENT, "forest tree " + std::to_string(k) + " has class " + std::to_string(c) +
                                    " >= n_classes " + std::to_string(n_classes));
      }
      total += sizes[k];
    }
    f->max_attribute = maxattr;
    uint32_t maxn = 0;
    for (uint32_t k = 0; k < t; ++k) maxn = std::max(maxn, sizes[k]);
    if (!compact_fits(maxn, maxattr, &f->abits) || total >= (1ull << 32))
      fail(ST_ERR_ARGUMENT, "forest too large for the compact device format");
    f->compact.reserve(total + t);
    for (uint32_t k = 0; k < t; ++k) {
      if (f->compact.size() & 1u) f->compact.push_back(CNode{0.0f, kLeafBit});  // 16-byte align
      f->offsets.push_back((uint32_t)f->compact.size());
      const uint32_t tb = (uint32_t)((sizes[k] * sizeof(CNode) + 15) & ~size_t(15));
      f->tree_bytes.push_back(tb);
      f->max_tree_bytes = std::max(f->max_tree_bytes, tb);
      for (uint32_t i = 0; i < sizes[k]; ++i) {
        const st_node& nd = trees[k][i];
        if (nd.class_id != ST_NO_CLASS)
          f->compact.push_back(CNode{nd.threshold, kLeafBit | nd.class_id});
        else
          f->compact.push_back(CNode{nd.threshold, ((8u * nd.child) << f->abits) | (4u * nd.attribute)});
      }
    }
    if (f->compact.size() & 1u) f->compact.push_back(CNode{0.0f, kLeafBit});
    f->compact.push_back(CNode{0.0f, kLeafBit});  // tail padding for the last 16-byte copy
    f->offsets.push_back((uint32_t)f->compact.size());
    *out = f.release();
  });
}

void st_forest_destroy(st_forest* forest) { delete forest; }

int st_eval_device(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                   int layout, const st_geom* geom, uint32_t* labels, st_stats* stats,
                   void* stream) {
  return guarded([&] {
    g_launches = 0;
    eval_device_impl(const_cast<st_tree*>(tree), x, m, a, ld, layout, geom, labels, stats,
                     static_cast<cudaStream_t>(stream));
  });
}

int st_eval(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
            const st_geom* geom, uint32_t* labels, st_stats* stats) {
  return guarded([&] {
    g_launches = 0;
    st_tree* t = const_cast<st_tree*>(tree);
    if (!t) fail(ST_ERR_ARGUMENT, "null tree");
    uint64_t ld2 = ld;
    check_common(m, a, ld2, layout, t->info.max_attribute);
    st_geom g{};
    if (geom) g = *geom;
    resolve_algo(t, g, stats != nullptr);
    if (m == 0) return;
    if (!x || !labels) fail(ST_ERR_ARGUMENT, "null data or label pointer");
    current_device();
    std::vector<std::pair<uint32_t*, uint32_t*>> extra;
    if (stats) {
      if (!stats->iterations || !stats->doubling_steps)
        fail(ST_ERR_ARGUMENT, "st_stats requires both arrays");
      extra.push_back({stats->iterations, nullptr});
      extra.push_back({stats->doubling_steps, nullptr});
    }
    uint32_t launches = 0;
    host_pipeline(x, m, a, ld2, layout, labels, extra,
                  [&](const float* xd, uint64_t rows, uint64_t ldd, uint32_t* lab,
                      std::vector<uint32_t*>& ex, cudaStream_t s) {
                    st_stats sd{};
                    if (stats) {
                      sd.iterations = ex[0];
                      sd.doubling_steps = ex[1];
                    }
                    eval_device_impl(t, xd, rows, a, ldd, layout, &g, lab, stats ? &sd : nullptr, s);
                    launches += g_launches;
                    g_launches = 0;
                  });
    g_launches = launches;
  });
}

int st_eval_timed(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                  int layout, const st_geom* geom, uint32_t* labels, st_timing* timing) {
  return guarded([&] {
    g_launches = 0;
    using Clock = std::chrono::steady_clock;
    auto us = [](Clock::duration d) { return std::chrono::duration<double, std::micro>(d).count(); };
    st_tree* t = const_cast<st_tree*>(tree);
    if (!t) fail(ST_ERR_ARGUMENT, "null tree");
    if (!timing) fail(ST_ERR_ARGUMENT, "null timing output");
    uint64_t ld2 = ld;
    check_common(m, a, ld2, layout, t->info.max_attribute);
    st_geom g{};
    if (geom) g = *geom;
    resolve_algo(t, g, false);
    *timing = st_timing{};
    if (m == 0) return;
    if (!x || !labels) fail(ST_ERR_ARGUMENT, "null data or label pointer");
    current_device();
    t->device(current_device());  // device replica outside the timed windows
    struct Ev {
      cudaStream_t s = nullptr;
      cudaEvent_t e[4] = {};
      ~Ev() {
        for (auto& x : e)
          if (x) cudaEventDestroy(x);
        if (s) cudaStreamDestroy(s);
      }
    } ev;
    CK(cudaStreamCreateWithFlags(&ev.s, cudaStreamNonBlocking));
    for (auto& e : ev.e) CK(cudaEventCreate(&e));
    const uint64_t row_bytes = (uint64_t)a * 4;
    const auto o0 = Clock::now();
    float* xd = nullptr;
    uint32_t* ld_out = nullptr;
    CK(cudaMalloc(&xd, m * row_bytes));
    struct Free {
      void* p[2];
      ~Free() {
        for (void* q : p)
          if (q) cudaFree(q);
      }
    } guard{{xd, nullptr}};
    CK(cudaMalloc(&ld_out, m * 4));
    guard.p[1] = ld_out;
    const auto a1 = Clock::now();
    CK(cudaEventRecord(ev.e[0], ev.s));
    if (layout == ST_LAYOUT_AOS) {
      if (ld2 == a)
        CK(cudaMemcpyAsync(xd, x, m * row_bytes, cudaMemcpyDefault, ev.s));
      else
        CK(cudaMemcpy2DAsync(xd, row_bytes, x, ld2 * 4, row_bytes, m, cudaMemcpyDefault, ev.s));
    } else {
      CK(cudaMemcpy2DAsync(xd, m * 4, x, ld2 * 4, m * 4, a, cudaMemcpyDefault, ev.s));
    }
    CK(cudaEventRecord(ev.e[1], ev.s));
    eval_device_impl(t, xd, m, a, layout == ST_LAYOUT_AOS ? (uint64_t)a : m, layout, &g, ld_out,
                     nullptr, ev.s);
    CK(cudaEventRecord(ev.e[2], ev.s));
    CK(cudaMemcpyAsync(labels, ld_out, m * 4, cudaMemcpyDefault, ev.s));
    CK(cudaEventRecord(ev.e[3], ev.s));
    CK(cudaStreamSynchronize(ev.s));
    const auto f0 = Clock::now();
    guard.p[0] = guard.p[1] = nullptr;
    CK(cudaFree(xd));
    CK(cudaFree(ld_out));
    const auto o1 = Clock::now();
    float ms[3];
    for (int k = 0; k < 3; ++k) CK(cudaEventElapsedTime(&ms[k], ev.e[k], ev.e[k + 1]));
    timing->outer_us = us(o1 - o0);
    timing->alloc_us = us(a1 - o0) + us(o1 - f0);
    timing->h2d_us = 1e3 * ms[0];
    timing->inner_us = 1e3 * ms[1];
    timing->d2h_us = 1e3 * ms[2];
  });
}

int st_forest_eval_device(const st_forest* forest, const float* x, uint64_t m, uint32_t a,
                          uint64_t ld, int layout, uint32_t* labels, void* stream) {
  return guarded([&] {
    g_launches = 0;
    forest_device_impl(const_cast<st_forest*>(forest), x, m, a, ld, layout, labels,
                       static_cast<cudaStream_t>(stream));
  });
}

int st_forest_eval(const st_forest* forest, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                   int layout, uint32_t* labels) {
  return guarded([&] {
    g_launches = 0;
    st_forest* f = const_cast<st_forest*>(forest);
    if (!f) fail(ST_ERR_ARGUMENT, "null forest");
    uint64_t ld2 = ld;
    check_common(m, a, ld2, layout, f->max_attribute);
    if (m == 0) return;
    if (!x || !labels) fail(ST_ERR_ARGUMENT, "null data or label pointer");
    current_device();
    uint32_t launches = 0;
    host_pipeline(x, m, a, ld2, layout, labels, {},
                  [&](const float* xd, uint64_t rows, uint64_t ldd, uint32_t* lab,
                      std::vector<uint32_t*>&, cudaStream_t s) {
                    forest_device_impl(f, xd, rows, a, ldd, layout, lab, s);
                    launches += g_launches;
                    g_launches = 0;
                  });
    g_launches = launches;
  });
}

int st_eval_sharded(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                    int layout, const st_geom* geom, const int* devices, int ndev,
                    uint32_t* labels) {
  return guarded([&] {
    g_launches = 0;
    st_tree* t = const_cast<st_tree*>(tree);
    if (!t) fail(ST_ERR_ARGUMENT, "null tree");
    if (ndev <= 0 || !devices) fail(ST_ERR_ARGUMENT, "ndev must be >= 1 with a device list");
    uint64_t ld2 = ld;
    check_common(m, a, ld2, layout, t->info.max_attribute);
    if (m == 0) return;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      fail(ST_ERR_NO_DEVICE, "no CUDA device available (no CPU fallback)");
    for (int k = 0; k < ndev; ++k)
      if (devices[k] < 0 || devices[k] >= count)
        fail(ST_ERR_ARGUMENT, "device id " + std::to_string(devices[k]) + " out of range");
    std::vector<int> rc(ndev, 0);
    std::vector<std::string> msg(ndev);
    std::vector<uint32_t> launches(ndev, 0);
    std::vector<std::thread> th;
    for (int k = 0; k < ndev; ++k) {
      th.emplace_back([&, k] {
        // Proc. 3 ranges: shard k owns [floor(k m / n), floor((k+1) m / n))
        const uint64_t lo = (uint64_t)((unsigned __int128)m * k / ndev);
        const uint64_t hi = (uint64_t)((unsigned __int128)m * (k + 1) / ndev);
        if (hi <= lo) return;
        if (cudaSetDevice(devices[k]) != cudaSuccess) {
          rc[k] = ST_ERR_CUDA;
          msg[k] = "cudaSetDevice failed";
          return;
        }
        const float* xs = layout == ST_LAYOUT_AOS ? x + lo * ld2 : x + lo;
        rc[k] = st_eval(t, xs, hi - lo, a, ld2, layout, geom, labels + lo, nullptr);
        if (rc[k]) msg[k] = st_last_error();
        launches[k] = st_last_launch_count();
      });
    }
    for (auto& h : th) h.join();
    uint32_t total = 0;
    for (int k = 0; k < ndev; ++k) {
      if (rc[k]) fail(rc[k], "shard " + std::to_string(k) + ": " + msg[k]);
      total += launches[k];
    }
    g_launches = total;
  });
}

}  // extern "C"

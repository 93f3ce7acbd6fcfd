// Internal host-side declarations shared by the C-ABI translation units
// (st_capi.cu: C ABI + host pipeline; st_data.cu / st_spec.cu / st_forest.cu:
// kernel dispatch, one kernel family per file so nvcc compiles them in
// parallel).  Not part of the public boundary (include/spectree_b200.h).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <deque>
#include <functional>
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
static_assert(sizeof(st_geom) == 96, "st_geom is part of the ABI (24 uint32 fields)");
static_assert(offsetof(st_node, attribute) == 0 && offsetof(st_node, threshold) == 4 &&
                  offsetof(st_node, child) == 8 && offsetof(st_node, class_id) == 12,
              "st_node field offsets must match spectree::EncodedNode");

namespace sti {


extern thread_local std::string g_error;  // st_capi.cu
extern thread_local uint32_t g_launches;

struct StError {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, std::string msg) { throw StError{code, std::move(msg)}; }

inline void cuda_check(cudaError_t e, const char* what) {
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
#define CK(x) ::sti::cuda_check((x), #x)

template <class F>
inline int guarded(F&& f) {
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

inline uint32_t ceil_log2(uint32_t v) {
  uint32_t s = 0, reach = 1;
  while (reach < v) {
    reach *= 2;
    ++s;
  }
  return s;
}

inline int current_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) fail(ST_ERR_NO_DEVICE, "no CUDA device available (no CPU fallback)");
  int d = 0;
  CK(cudaGetDevice(&d));
  return d;
}

// Table uploads (tree nodes, window tables, forests).  They are read by
// kernels on the caller's streams, which may be non-blocking: a cudaMemcpy
// from pageable memory may return before its DMA has landed, and a
// non-blocking stream does not order behind the legacy stream -- so every
// upload is enqueued on the legacy stream and that stream is drained
// (publish) before the device pointer is handed out.
inline void upload(void* dst, const void* src, size_t bytes) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cudaStreamLegacy));
}
inline void zero_fill(void* dst, size_t bytes) { CK(cudaMemsetAsync(dst, 0, bytes, cudaStreamLegacy)); }
inline void publish() { CK(cudaStreamSynchronize(cudaStreamLegacy)); }

struct DevProps {
  int sms = 0;
  size_t smem_optin = 0;
  size_t smem_per_sm = 0;
};
inline DevProps dev_props(int dev) {
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
  // One-window trees: entries[pm_off + j] = path mask of leaf j
  // {thr = 0, attr_steps = leaf code, left = care, right = want}: bits of the
  // window lanes on the root-to-leaf path and their right-turn directions.
  // Unused lanes carry code 0.  pm_off 0 = none (more windows, more leaves
  // than lanes, or a DAG-shaped input).
  uint32_t pm_off = 0;
  // 8-byte windows (k_spec_ring CW), appended as SEntry units at cw_off
  // (cw_units of them; 0 = none): entry (w, j) at 8 * (G * w + j) bytes,
  // word = attr4 | left << cw_abits | right << (cw_abits + cw_cbits).
  uint32_t cw_off = 0, cw_units = 0, cw_abits = 0, cw_cbits = 0;
  // Self-loop 8-byte windows (k_spec_ring SL), appended at sl_off (sl_units
  // SEntry units; 0 = none): entry (w, j) at 8 * (G * w + j), word = attr4 |
  // left << sl_abits | right << (sl_abits + sl_cbits).  A code is a lane
  // target t < G, or payload << log2(G) | j for a terminal -- payload = the
  // next window (>= 1; nothing exits to the root window) or sl_nw + leaf
  // code -- so a terminal's low bits name its own lane and a width-G shfl
  // pointer-jumping step returns it unchanged (no select per step), and
  // (payload << log2 G) * 8 is the next window's byte offset.  Windows
  // sl_nw.. hold copies of window 0: after a leaf the stream restarts at the
  // root without a select.
  uint32_t sl_off = 0, sl_units = 0, sl_abits = 0, sl_cbits = 0, sl_nw = 0;
  // fixed-trip loop: the most windows any record visits, and the expected
  // count under the synthetic data distribution (leaf weight 2^-depth)
  uint32_t sl_wmax = 0;
  double sl_wmean = 0.0;
  uint32_t sl_ws = 0;  // entries per window in the self-loop table
  // One-window trees: entries[sl1_off + j] = {thr, 4*attr, left, right} with
  // self-loop leaf codes kLeafBit | leaf code << 5 | j (0 = none).
  uint32_t sl1_off = 0;
  uint32_t base_units = 0;  // entries of the 16-byte table incl. path masks (cw / sl tables follow)
};

}  // namespace sti
using namespace sti;  // st_tree / st_forest below are the C ABI's opaque structs (global)

struct st_tree {
  std::vector<st_node> nodes;
  st_tree_info info{};
  uint32_t abits = 1;
  bool compact_ok = true;
  bool leaf_table = false;            // some class >= 2^30: leaves carry ordinals
  std::vector<uint32_t> leaf_classes;  // ordinal -> class
  std::vector<uint32_t> leaf_code;     // node -> code payload (class or ordinal)
  std::vector<CNode> compact;
  std::vector<CNode> folded;  // leaf pairs folded into terminals (data walk, shared tree)
  bool fold_ok = false;

  std::mutex mu;
  std::map<std::pair<uint32_t, uint32_t>, std::shared_ptr<WinTable>> wins;  // (G, H)
  struct Dev {
    CNode* compact = nullptr;
    CNode* folded = nullptr;
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
      cudaFree(kv.second.folded);
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
      wt.base_units = 32;
      return wt;
    }
    std::vector<int32_t> win_of_root(n, -1);
    std::vector<std::vector<uint32_t>> members;
    std::vector<std::vector<uint32_t>> ldepth;
    std::vector<uint32_t> wdepth{1};  // windows on the path from the root window, inclusive
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
          wdepth.push_back(wdepth[w] + 1);
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
    // 8-byte windows if every field fits: attr4 in abits, codes in cbits =
    // (32 - abits) / 2 with (cbits - 2)-bit window indices and classes
    uint32_t max_a4 = 0, max_code = 0;
    for (uint32_t i = 0; i < n; ++i) {
      if (is_leaf(i)) max_code = std::max(max_code, leaf_code[i]);
      else max_a4 = std::max(max_a4, 4u * nodes[i].attribute);
    }
    uint32_t abits = 2;
    while ((max_a4 >> abits) != 0) ++abits;
    const uint32_t cbits = (32 - abits) / 2;
    const bool cw = G <= 32 && cbits >= 8 && nw < (1u << (cbits - 2)) && max_code < (1u << (cbits - 2)) &&
                    (uint64_t)nw * G < (1u << 24);
    std::vector<uint2> cwt;
    if (cw) cwt.assign((size_t)nw * G + 64, make_uint2(0u, 0u));
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
      auto ccode = [&](uint32_t c) -> uint32_t {
        if (is_leaf(c)) return (1u << (cbits - 1)) | leaf_code[c];
        if (lane_of[c] >= 0) return (uint32_t)lane_of[c];
        return (1u << (cbits - 2)) | (uint32_t)win_of_root[c];
      };
      for (uint32_t j = 0; j < mem.size(); ++j) {
        const st_node& nd = nodes[mem[j]];
        SEntry e;
        e.thr = nd.threshold;
        e.attr_steps = (4u * nd.attribute) | (steps << 24);
        e.left = code(nd.child);
        e.right = code(nd.child + 1);
        wt.entries[base[w] + j] = e;
        if (cw) {
          uint32_t tb;
          std::memcpy(&tb, &nd.threshold, 4);
          cwt[(size_t)w * G + j] = make_uint2(
              tb, (4u * nd.attribute) | (ccode(nd.child) << abits) | (ccode(nd.child + 1) << (abits + cbits)));
        }
      }
      // unused lanes of the window read the window root's attribute (code 0:
      // they point at lane 0, never on a path): the same shared-memory word
      // as lane 0 -- a broadcast, not an extra bank conflict
      if (cw)
        for (uint32_t j = (uint32_t)mem.size(); j < G; ++j)
          cwt[(size_t)w * G + j] = make_uint2(0u, 4u * nodes[mem[0]].attribute);
      for (uint32_t j = 0; j < mem.size(); ++j) lane_of[mem[j]] = -1;
    }
    wt.root_code = kExitBit | 0u;
    wt.windows = nw;
    if (nw == 1) {
      add_path_masks(wt, members[0], G);
      // one-window self-loop entries: leaf codes kLeafBit | code << 5 | j
      if (max_code < (1u << 26)) {
        const auto& mem = members[0];
        std::vector<SEntry> s1(32, SEntry{0.0f, 0u, 0u, 0u});
        for (uint32_t j = 0; j < mem.size(); ++j) lane_of[mem[j]] = (int32_t)j;
        for (uint32_t j = 0; j < mem.size(); ++j) {
          auto code = [&](uint32_t c) -> uint32_t {
            if (is_leaf(c)) return kLeafBit | (leaf_code[c] << 5) | j;
            return (uint32_t)lane_of[c];
          };
          const st_node& nd = nodes[mem[j]];
          s1[j] = SEntry{nd.threshold, 4u * nd.attribute, code(nd.child), code(nd.child + 1)};
        }
        wt.sl1_off = (uint32_t)wt.entries.size();
        wt.entries.insert(wt.entries.end(), s1.begin(), s1.end());
      }
    }
    // the 16-byte-entry kernels stage [0, base_units): windows, path masks
    wt.base_units = (uint32_t)wt.entries.size();
    if (cw) {
      if (cwt.size() & 1) cwt.push_back(make_uint2(0u, 0u));
      wt.cw_off = (uint32_t)wt.entries.size();
      wt.cw_units = (uint32_t)(cwt.size() / 2);
      wt.cw_abits = abits;
      wt.cw_cbits = cbits;
      const size_t base_units = wt.entries.size();
      wt.entries.resize(base_units + wt.cw_units, SEntry{0.0f, 0u, 0u, 0u});
      std::memcpy(wt.entries.data() + base_units, cwt.data(), cwt.size() * sizeof(uint2));
    }
    // self-loop 8-byte windows (see WinTable): codes of cbits2 bits
    {
      uint32_t lg = 0;
      while ((1u << lg) < G) ++lg;
      const uint64_t ncodes = (uint64_t)max_code + 1;  // leaf payloads sl_nw + code
      const uint64_t units = (uint64_t)nw + ncodes;      // windows + root copies
      uint32_t cbits2 = 1;
      while (cbits2 < 40 && ((units * G - 1) >> cbits2) != 0) ++cbits2;
      // ws entries per window (the largest window; lanes >= ws read lane
      // 0's entry): G = 4 two-level windows pack their 3 nodes in 24 B
      uint32_t ws = 1;
      for (uint32_t w = 0; w < nw; ++w) ws = std::max<uint32_t>(ws, (uint32_t)members[w].size());
      if ((8u * ws) % G != 0) ws = G;
      // (codes fit 16 bits: the kernels broadcast two streams' codes in one word)
      if (G <= 32 && (1u << lg) == G && ncodes <= 64 && abits + 2 * cbits2 <= 32 && cbits2 <= 16 &&
          units * G < (1u << 24)) {
        std::vector<uint2> slt((size_t)units * ws + 64, make_uint2(0u, 0u));
        for (uint32_t w = 0; w < nw; ++w) {
          const auto& mem = members[w];
          for (uint32_t j = 0; j < mem.size(); ++j) lane_of[mem[j]] = (int32_t)j;
          for (uint32_t j = 0; j < mem.size(); ++j) {
            auto scode = [&](uint32_t c) -> uint32_t {
              if (is_leaf(c)) return ((nw + leaf_code[c]) << lg) | j;
              if (lane_of[c] >= 0) return (uint32_t)lane_of[c];
              return ((uint32_t)win_of_root[c] << lg) | j;
            };
            const st_node& nd = nodes[mem[j]];
            uint32_t tb;
            std::memcpy(&tb, &nd.threshold, 4);
            slt[(size_t)w * ws + j] = make_uint2(
                tb, (4u * nd.attribute) | (scode(nd.child) << abits) | (scode(nd.child + 1) << (abits + cbits2)));
          }
          for (uint32_t j = (uint32_t)mem.size(); j < ws; ++j)  // unused lanes: the root's word (broadcast)
            slt[(size_t)w * ws + j] = make_uint2(0u, 4u * nodes[mem[0]].attribute);
          for (uint32_t j = 0; j < mem.size(); ++j) lane_of[mem[j]] = -1;
        }
        // Leaf sinks: window sl_nw + c holds, in every lane, the terminal
        // code of leaf payload c on both sides, so a stream that reached a
        // leaf stays there for any number of further window steps (leaves
        // are fixpoints, eval_speculative.cpp:38-51) -- the fixed-trip loop
        // runs every record for sl_wmax steps with no per-step test.
        for (uint64_t w = nw; w < units; ++w)
          for (uint32_t j = 0; j < ws; ++j) {
            const uint32_t code = ((uint32_t)w << lg) | j;
            slt[(size_t)w * ws + j] = make_uint2(0u, (code << abits) | (code << (abits + cbits2)));
          }
        if (slt.size() & 1) slt.push_back(make_uint2(0u, 0u));
        wt.sl_off = (uint32_t)wt.entries.size();
        wt.sl_units = (uint32_t)(slt.size() / 2);
        wt.sl_abits = abits;
        wt.sl_cbits = cbits2;
        wt.sl_nw = nw;
        wt.sl_ws = ws;
        // fixed-trip statistics: the deepest window count, and its mean over
        // records under uniform data and midpoint splits (leaf weight
        // 2^-depth: the synthetic generators' volume fractions)
        std::vector<uint32_t> nd(n, 0);
        double ew = 0.0, wsum = 0.0;
        for (uint32_t i = 0; i < n; ++i) {
          if (is_leaf(i)) continue;
          for (uint32_t c : {nodes[i].child, nodes[i].child + 1}) nd[c] = std::max(nd[c], nd[i] + 1);
        }
        std::vector<uint32_t> win_of_node(n, 0);
        for (uint32_t w = 0; w < nw; ++w)
          for (uint32_t u : members[w]) win_of_node[u] = w;
        for (uint32_t i = 0; i < n; ++i) {
          if (is_leaf(i)) continue;
          for (uint32_t c : {nodes[i].child, nodes[i].child + 1}) {
            if (!is_leaf(c)) continue;
            const double wt_c = std::ldexp(1.0, -(int)std::min<uint32_t>(nd[c], 1000));
            wsum += wt_c;
            ew += wt_c * wdepth[win_of_node[i]];
          }
        }
        wt.sl_wmax = *std::max_element(wdepth.begin(), wdepth.end());
        wt.sl_wmean = wsum > 0 ? ew / wsum : (double)wt.sl_wmax;
        wt.entries.resize(wt.entries.size() + wt.sl_units, SEntry{0.0f, 0u, 0u, 0u});
        std::memcpy(wt.entries.data() + wt.sl_off, slt.data(), slt.size() * sizeof(uint2));
      }
    }
    return wt;
  }

  // Path masks of a one-window tree (ballot reduction, k_spec_ring SR == 0):
  // leaf l is reached iff ((preds ^ want_l) & care_l) == 0, preds = the
  // window lanes' predicate bits (1 = right, the reference's x > thr).
  void add_path_masks(WinTable& wt, const std::vector<uint32_t>& mem, uint32_t G) const {
    if (mem.size() > 32) return;
    std::vector<int32_t> lane_of(nodes.size(), -1);
    for (uint32_t j = 0; j < mem.size(); ++j) lane_of[mem[j]] = (int32_t)j;
    std::vector<uint8_t> seen(nodes.size(), 0);
    std::vector<SEntry> pm;
    struct Item { uint32_t node, care, want; };
    std::vector<Item> stack{{0u, 0u, 0u}};
    while (!stack.empty()) {
      const Item it = stack.back();
      stack.pop_back();
      if (seen[it.node]++) return;  // reached twice: DAG-shaped input
      if (is_leaf(it.node)) {
        pm.push_back(SEntry{0.0f, kLeafBit | leaf_code[it.node], it.care, it.want});
        continue;
      }
      const int32_t j = lane_of[it.node];
      if (j < 0) return;
      const uint32_t bit = 1u << j;
      stack.push_back({nodes[it.node].child, it.care | bit, it.want});
      stack.push_back({nodes[it.node].child + 1, it.care | bit, it.want | bit});
    }
    if (pm.size() > G) return;
    wt.pm_off = (uint32_t)wt.entries.size();
    pm.resize(32, SEntry{0.0f, 0u, 0u, 0u});  // unused lanes: code 0, never stored
    wt.entries.insert(wt.entries.end(), pm.begin(), pm.end());
  }

  Dev& device(int d) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = dev.find(d);
    if (it != dev.end()) return it->second;
    Dev dv;
    CK(cudaMalloc(&dv.wide, nodes.size() * sizeof(st_node)));
    upload(dv.wide, nodes.data(), nodes.size() * sizeof(st_node));
    if (compact_ok) {
      const size_t bytes = ((compact.size() * sizeof(CNode) + 15) & ~size_t(15)) + 16;
      CK(cudaMalloc(&dv.compact, bytes));
      zero_fill(dv.compact, bytes);
      upload(dv.compact, compact.data(), compact.size() * sizeof(CNode));
    }
    if (fold_ok) {
      const size_t bytes = ((folded.size() * sizeof(CNode) + 15) & ~size_t(15)) + 16;
      CK(cudaMalloc(&dv.folded, bytes));
      zero_fill(dv.folded, bytes);
      upload(dv.folded, folded.data(), folded.size() * sizeof(CNode));
    }
    std::vector<uint32_t> map;  // lives until publish()
    for (uint32_t i = 0; i < nodes.size(); ++i)
      if (!is_leaf(i)) map.push_back(i);
    map.push_back(0);  // keep the allocation non-empty
    CK(cudaMalloc(&dv.internal_map, map.size() * 4));
    upload(dv.internal_map, map.data(), map.size() * 4);
    if (leaf_table) {
      CK(cudaMalloc(&dv.leaf_tbl, leaf_classes.size() * 4));
      upload(dv.leaf_tbl, leaf_classes.data(), leaf_classes.size() * 4);
    }
    publish();
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
    upload(p, wt.entries.data(), wt.entries.size() * sizeof(SEntry));
    publish();
    dv.wins[key] = p;
    return p;
  }
};

struct st_forest {
  // Two node layouts of the same trees: [0] folded where the encoding allows
  // (leaf pairs inside terminal nodes, fold_tree; the default), [1] plain
  // compact nodes (ST_VAR_NO_FOLD).  Labels are identical.
  struct Layout {
    std::vector<CNode> compact;        // trees concatenated, each starting 16-byte aligned
    std::vector<uint32_t> offsets;     // first node of each tree (+ end sentinel)
    std::vector<uint32_t> tree_bytes;  // bytes per tree rounded up to 16 (bulk-copy size)
    uint32_t max_tree_bytes = 0;
  } lay[2];
  uint32_t t_count = 0, n_classes = 0, abits = 1, max_attribute = 0;
  std::mutex mu;
  struct Dev {
    CNode* nodes = nullptr;
    uint32_t* offsets = nullptr;
    uint32_t* tree_bytes = nullptr;
  };
  std::map<std::pair<int, int>, Dev> dev;  // (device, layout)
  ~st_forest() {
    int cur = -1;
    cudaGetDevice(&cur);
    for (auto& kv : dev) {
      if (cudaSetDevice(kv.first.first) != cudaSuccess) continue;
      cudaFree(kv.second.nodes);
      cudaFree(kv.second.offsets);
      cudaFree(kv.second.tree_bytes);
    }
    if (cur >= 0) cudaSetDevice(cur);
  }
  Dev& device(int d, int l) {
    std::lock_guard<std::mutex> lk(mu);
    auto it = dev.find({d, l});
    if (it != dev.end()) return it->second;
    const Layout& L = lay[l];
    Dev dv;
    CK(cudaMalloc(&dv.nodes, L.compact.size() * sizeof(CNode) + 16));
    upload(dv.nodes, L.compact.data(), L.compact.size() * sizeof(CNode));
    CK(cudaMalloc(&dv.offsets, L.offsets.size() * 4));
    upload(dv.offsets, L.offsets.data(), L.offsets.size() * 4);
    CK(cudaMalloc(&dv.tree_bytes, L.tree_bytes.size() * 4));
    upload(dv.tree_bytes, L.tree_bytes.data(), L.tree_bytes.size() * 4);
    publish();
    return dev.emplace(std::make_pair(d, l), dv).first->second;
  }
};

namespace sti {

// ---------------------------------------------------------------------------
// Tree construction
// ---------------------------------------------------------------------------
inline void validate_links(const st_node* nodes, uint32_t n, const char* what) {
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

inline uint32_t bits_for(uint64_t v) {  // bits to hold values 0..v
  uint32_t b = 1;
  while (b < 64 && (v >> b) != 0) ++b;
  return b;
}

// Compact meta for an internal node: (8*child) << abits | 4*attr.
inline bool compact_fits(uint32_t n, uint32_t max_attribute, uint32_t* abits) {
  // at least 6 bits: the register walk selects x[attr] from the meta's bits
  // 2..5 (16 attributes) without masking, so they must be attribute bits
  *abits = std::max<uint32_t>(6, bits_for(4ull * max_attribute));
  return *abits < 31 && ((8ull * n) << *abits) < (1ull << 31);
}

// Folded compact layout: BFS, children adjacent, every internal node whose two
// children are leaves becomes a terminal {thr, kLeafBit | kPairBit | classR <<
// 20 | classL << 10 | 4*attr} and its leaf pair is dropped (classes < 1024,
// 4*attr < 1024 are the caller's preconditions).  False when the folded array
// would not shrink (DAG-shaped inputs) or not fit the compact child field.
inline bool fold_tree(const st_node* nodes, uint32_t n, uint32_t abits, std::vector<CNode>& f) {
  auto is_leaf = [&](uint32_t i) { return nodes[i].class_id != ST_NO_CLASS; };
  std::vector<uint32_t> order{0};  // original index per folded slot
  f.clear();
  for (size_t k = 0; k < order.size() && order.size() <= 2ull * n; ++k) {
    const st_node& nd = nodes[order[k]];
    if (is_leaf(order[k])) {
      f.push_back(CNode{nd.threshold, kLeafBit | nd.class_id});
    } else if (is_leaf(nd.child) && is_leaf(nd.child + 1)) {
      f.push_back(CNode{nd.threshold, kLeafBit | kPairBit | (nodes[nd.child + 1].class_id << 20) |
                                          (nodes[nd.child].class_id << 10) | (4u * nd.attribute)});
    } else {
      const uint32_t fc = (uint32_t)order.size();  // children take the next two slots
      f.push_back(CNode{nd.threshold, ((8u * fc) << abits) | (4u * nd.attribute)});
      order.push_back(nd.child);
      order.push_back(nd.child + 1);
    }
  }
  return f.size() == order.size() && f.size() <= n && ((8ull * f.size()) << abits) < (1ull << 31);
}

inline std::unique_ptr<st_tree> make_tree(const st_node* nodes, uint32_t n) {
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
      // classes >= 2^30 would collide with the folded-terminal marker
      // (kPairBit) in the inline leaf encoding: leaves then carry ordinals
      // into a class table instead
      if (nd.class_id >= kPairBit) t->leaf_table = true;
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
  // Folded layout for the shared-tree data walk (fold_tree)
  if (t->compact_ok && !t->leaf_table && in.max_class < 1024 && 4ull * in.max_attribute < 1024 && n > 1)
    t->fold_ok = fold_tree(nodes, n, t->abits, t->folded);
  return t;
}

// ---------------------------------------------------------------------------
// Launch helpers
// ---------------------------------------------------------------------------
inline int blocks_for(const void* fn, size_t smem, int dev, uint32_t blocks_per_sm, uint64_t n_tiles,
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
inline void clear_stale_error() { (void)cudaGetLastError(); }

inline void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(ST_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  ++g_launches;
}

inline void check_common(uint64_t m, uint32_t a, uint64_t& ld, int layout, uint32_t max_attribute) {
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

inline EncodeTiledFn encode_tiled() {
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

inline uint32_t round1024(uint64_t b) { return (uint32_t)((b + 1023) & ~uint64_t(1023)); }

// TMA applies to packed AoS, 16 B-aligned, with a tile of <= 256 rows of 32 floats.
inline bool tma_ok(const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout, uint32_t S) {
  if (layout != ST_LAYOUT_AOS || ld != a) return false;
  if ((reinterpret_cast<uintptr_t>(x) & 15u) != 0) return false;
  if (32ull * S * a > 8192) return false;         // box rows = 32*S*a/32 <= 256
  if (m < 32ull * S) return false;                 // no full tile: nothing for TMA to move
  if (m * (uint64_t)a / 32 >= (1ull << 31)) return false;
  return encode_tiled() != nullptr;
}

// box rows = one tile of 32*S records, or `records` (a multiple of 32 / a)
inline void make_tmap(Staging& st, const float* x, uint64_t m, uint32_t a, uint32_t records = 0) {
  const cuuint64_t dims[2] = {32, (cuuint64_t)(m * (uint64_t)a / 32)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {32, (records ? records : 32u * st.S) * a / 32u};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_tiled()(&st.tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x),
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
}

// Choose loader, S and stages.  `fixed` = shared bytes needed besides the
// record stages (tree / windows / counters).
inline Staging plan_staging(const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout, uint32_t S,
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

inline uint32_t pick_warps(uint32_t want, const Staging& st, size_t fixed, const DevProps& pr) {
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
inline uint32_t default_bps(uint32_t want, const Staging& st, uint64_t m, const DevProps& pr) {
  if (want) return want;
  if (st.loader != kTma) return 0;
  // one wide CTA per SM carries the ~128 KB of stages (pick_warps); more CTAs
  // only pay on inputs too small to fill the SMs
  const uint64_t tiles = m / (32ull * st.S);
  return tiles >= (uint64_t)pr.sms * st.warps * 16 ? std::max<uint32_t>(1, 16 / st.warps) : 0u;
}

inline PipeArgs pipe_args(const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout) {
  PipeArgs p{};
  p.x = x;
  p.m = m;
  p.a = a;
  p.ld = (uint32_t)ld;
  p.layout_soa = layout == ST_LAYOUT_SOA ? 1u : 0u;
  return p;
}

// Compile-time arities with a TMA fast path; everything else runs A = 0.
inline bool ct_arity(uint32_t a) { return a == 8 || a == 16 || a == 32 || a == 64; }

// ---- cross-translation-unit entry points ------------------------------------
// Data-kernel launch plan (st_data.cu): staging, tree location, arguments.
struct DataPlan {
  Staging stg;
  int tloc = 0;
  DataArgs d{};
  size_t smem = 0;
  uint32_t bps = 0;
};
DataPlan plan_data(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                   const st_geom& g, uint32_t* labels, uint32_t* depths, int dev);
uint32_t choose_S(uint32_t a, uint32_t want, bool small);
void eval_data_device(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                      const st_geom& g, uint32_t* labels, uint32_t* depths, cudaStream_t s,
                      int dev);                                                         // st_data.cu
void spec_geometry(const st_tree* t, const st_geom& g, uint32_t& G, uint32_t& H);     // st_spec.cu
// frame-stream launch of the speculative ring (st_frames.cu -> st_spec.cu)
struct SpecFrames {
  uint32_t* fctl = nullptr;
  uint32_t ring = 0, max_ctas = 0;
  uint64_t ring_records = 0, idle_ns = 0;
  uint64_t tiles = 0;  // out: ring slots (tiles) per frame
};
void eval_spec_device(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                      const st_geom& g, uint32_t* labels, st_stats* stats, cudaStream_t s,
                      int dev, SpecFrames* fr = nullptr);                             // st_spec.cu
void forest_device_impl(st_forest* f, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                        int layout, const st_geom& g, uint32_t* labels, cudaStream_t s);  // st_forest.cu
}  // namespace sti

// spectree_b200.hpp -- header-only C++ drop-in over the C ABI, mirroring the
// reference evaluate API (/root/reference/proj/core) signature for signature.
//
// Include it inside the reference build (it uses the reference's own types and
// exceptions) and swap the evaluator call:
//
//   spectree::eval_data_parallel(tree, data, cfg)        eval_data_parallel.hpp:31-33
//     -> spectree_b200::eval_data_parallel(tree, data, cfg)
//   spectree::eval_speculative(tree, data, cfg, &stats)  eval_speculative.hpp:100-106
//     -> spectree_b200::eval_speculative(tree, data, cfg, &stats)
//   spectree::eval_speculative_basic(...)                eval_speculative.hpp:92-98
//     -> spectree_b200::eval_speculative_basic(...)
//
// Semantics kept: inputs are const references owned by the caller, the
// ClassAssignment is returned by value, geometry and attribute-range problems
// throw spectree::ArgumentError before any work with the reference's messages
// (validate_data_parallel / validate_speculative / check_attribute_range),
// empty datasets return an empty assignment, results never depend on the
// geometry.  CUDA failures throw spectree::Error; there is no CPU fallback.
#pragma once

#include <spectree/dataset.hpp>
#include <spectree/errors.hpp>
#include <spectree/eval_data_parallel.hpp>
#include <spectree/eval_serial.hpp>
#include <spectree/eval_speculative.hpp>
#include <spectree/tree.hpp>

#include <memory>
#include <string>
#include <vector>

#include "spectree_b200.h"

static_assert(sizeof(spectree::EncodedNode) == sizeof(st_node),
              "spectree::EncodedNode and st_node must be layout-identical");

namespace spectree_b200 {

/// GPU geometry on top of the reference configs (zero = automatic).
struct GpuConfig {
  st_geom geom{};
  std::vector<int> devices;  // > 1 entries: sample-sharded over these GPUs
};

namespace detail {

inline void check(int rc) {
  if (rc == ST_OK) return;
  const std::string msg = st_last_error();
  if (rc == ST_ERR_ARGUMENT) throw spectree::ArgumentError(msg);
  if (rc == ST_ERR_IO) throw spectree::IoError(msg);
  throw spectree::Error("spectree_b200: " + msg);
}

struct TreeDeleter {
  void operator()(st_tree* t) const { st_tree_destroy(t); }
};
using TreeHandle = std::unique_ptr<st_tree, TreeDeleter>;

inline TreeHandle make_handle(const spectree::EncodedTree& tree) {
  st_tree* t = nullptr;
  check(st_tree_create(reinterpret_cast<const st_node*>(tree.nodes().data()), tree.size(), &t));
  return TreeHandle(t);
}

inline spectree::ClassAssignment run(const spectree::EncodedTree& tree,
                                     const spectree::Dataset& data, st_geom geom,
                                     const GpuConfig& gpu, st_stats* stats) {
  spectree::check_attribute_range(tree, data);  // eval_serial.cpp:10-17, before any work
  spectree::ClassAssignment out(data.count());
  if (data.count() == 0) return out;
  TreeHandle h = make_handle(tree);
  if (gpu.devices.size() > 1 && stats == nullptr) {
    check(st_eval_sharded(h.get(), data.values().data(), data.count(), data.arity(), 0,
                          ST_LAYOUT_AOS, &geom, gpu.devices.data(), (int)gpu.devices.size(),
                          out.data()));
  } else {
    check(st_eval(h.get(), data.values().data(), data.count(), data.arity(), 0, ST_LAYOUT_AOS,
                  &geom, out.data(), stats));
  }
  return out;
}

inline uint32_t next_pow2(uint32_t v) {
  uint32_t p = 1;
  while (p < v) p *= 2;
  return p;
}

}  // namespace detail

/// Data decomposition (Algorithm 1): reference validation, GPU execution.
inline spectree::ClassAssignment eval_data_parallel(const spectree::EncodedTree& tree,
                                                    const spectree::Dataset& data,
                                                    const spectree::DataParallelConfig& config,
                                                    const GpuConfig& gpu = {}) {
  spectree::validate_data_parallel(config, data.count());  // eval_data_parallel.cpp:13-33
  st_geom g = gpu.geom;
  g.algo = ST_ALGO_DATA;
  return detail::run(tree, data, g, gpu, nullptr);
}

namespace detail {
inline spectree::ClassAssignment speculative(const spectree::EncodedTree& tree,
                                             const spectree::Dataset& data,
                                             const spectree::SpeculativeConfig& config,
                                             spectree::SpeculativeStats* stats, bool basic,
                                             const GpuConfig& gpu) {
  spectree::validate_speculative(config, tree, data.count(), basic);  // eval_speculative.cpp:69-107
  st_geom g = gpu.geom;
  g.algo = ST_ALGO_SPECULATIVE;
  const uint32_t internal = (tree.size() - 1) / 2;
  if (g.group_lanes == 0 && internal <= 32) g.group_lanes = next_pow2(internal ? internal : 1);
  std::vector<std::uint32_t> it, st;
  st_stats s{};
  if (stats) {
    // counters follow the barrier-separated law: k doublings per root check
    g.reductions = basic ? 1 : config.reductions_per_iteration;
    it.assign(data.count(), 0);
    st.assign(data.count(), 0);
    s.iterations = it.data();
    s.doubling_steps = st.data();
  }
  spectree::ClassAssignment out = run(tree, data, g, gpu, stats ? &s : nullptr);
  if (stats) {
    stats->iterations = std::move(it);
    stats->doubling_steps = std::move(st);
    stats->barriers = data.count();
    for (std::uint32_t v : stats->doubling_steps) stats->barriers += v;
  }
  return out;
}
}  // namespace detail

/// Mapped-lane speculative decomposition (Algorithm 2, paper Proc. 5).
inline spectree::ClassAssignment eval_speculative(const spectree::EncodedTree& tree,
                                                  const spectree::Dataset& data,
                                                  const spectree::SpeculativeConfig& config,
                                                  spectree::SpeculativeStats* stats = nullptr,
                                                  const GpuConfig& gpu = {}) {
  return detail::speculative(tree, data, config, stats, false, gpu);
}

/// All-lanes variant (paper Proc. 4).  Leaves are fixpoints, so the GPU
/// evaluates internal lanes only; labels and the k = 1 counters match.
inline spectree::ClassAssignment eval_speculative_basic(const spectree::EncodedTree& tree,
                                                        const spectree::Dataset& data,
                                                        const spectree::SpeculativeConfig& config,
                                                        spectree::SpeculativeStats* stats = nullptr,
                                                        const GpuConfig& gpu = {}) {
  return detail::speculative(tree, data, config, stats, true, gpu);
}

/// traversal_depths (eval_serial.hpp:23-25, eval_serial.cpp:77-97): root-to-leaf
/// edge count per record, computed on the GPU by the data kernel
/// (st_eval_depths).  Attribute range checked first, as the reference does.
inline std::vector<std::uint32_t> traversal_depths(const spectree::EncodedTree& tree,
                                                   const spectree::Dataset& data,
                                                   const GpuConfig& gpu = {}) {
  spectree::check_attribute_range(tree, data);
  std::vector<std::uint32_t> depths(data.count()), labels(data.count());
  if (data.count() == 0) return depths;
  detail::TreeHandle h = detail::make_handle(tree);
  detail::check(st_eval_depths(h.get(), data.values().data(), data.count(), data.arity(), 0,
                               ST_LAYOUT_AOS, &gpu.geom, labels.data(), depths.data()));
  return depths;
}

/// mean_traversal_depth (eval_serial.hpp:27-29, eval_serial.cpp:99-110): the
/// d_mu of the cost model; an empty dataset throws ArgumentError.
inline double mean_traversal_depth(const spectree::EncodedTree& tree, const spectree::Dataset& data,
                                   const GpuConfig& gpu = {}) {
  if (data.count() == 0) throw spectree::ArgumentError("mean traversal depth of an empty dataset");
  const auto depths = traversal_depths(tree, data, gpu);
  std::uint64_t total = 0;
  for (const std::uint32_t d : depths) total += d;
  return static_cast<double>(total) / static_cast<double>(depths.size());
}

/// Random forest with a per-record majority vote (smallest class id on ties).
inline spectree::ClassAssignment eval_forest(const std::vector<spectree::EncodedTree>& trees,
                                             const spectree::Dataset& data, uint32_t n_classes,
                                             const GpuConfig& gpu = {}) {
  std::vector<const st_node*> ptrs;
  std::vector<uint32_t> sizes;
  for (const auto& t : trees) {
    spectree::check_attribute_range(t, data);
    ptrs.push_back(reinterpret_cast<const st_node*>(t.nodes().data()));
    sizes.push_back(t.size());
  }
  st_forest* f = nullptr;
  detail::check(st_forest_create(ptrs.data(), sizes.data(), (uint32_t)trees.size(), n_classes, &f));
  std::unique_ptr<st_forest, void (*)(st_forest*)> guard(f, st_forest_destroy);
  spectree::ClassAssignment out(data.count());
  if (data.count())
    detail::check(st_forest_eval(f, data.values().data(), data.count(), data.arity(), 0,
                                 ST_LAYOUT_AOS, &gpu.geom, out.data()));
  return out;
}

/// Resident frame stream (st_frames_*): one data-decomposition grid stays on
/// the GPU and classifies frame after frame of `records` records (the C3
/// per-pixel workload) with no launch per frame.  push() copies a host frame
/// into the next ring slot and publishes it; pop(seq) waits for that frame's
/// labels (pop frame seq before pushing frame seq + ring).  Device producers
/// use slot() / acquire() / publish() / wait() on their own CUDA streams
/// (include/spectree_b200.h).  Labels equal eval_data_parallel's per frame.
class FrameStream {
 public:
  FrameStream(const spectree::EncodedTree& tree, std::uint64_t records, std::uint32_t arity,
              std::uint32_t ring = 4, const GpuConfig& gpu = {}, std::uint32_t idle_timeout_ms = 0)
      : tree_(detail::make_handle(tree)), records_(records) {
    st_geom g = gpu.geom;
    g.algo = ST_ALGO_DATA;
    detail::check(st_frames_open(tree_.get(), records, arity, ring, &g, 0, idle_timeout_ms, &f_));
  }
  FrameStream(const FrameStream&) = delete;
  FrameStream& operator=(const FrameStream&) = delete;
  ~FrameStream() {
    if (f_) st_frames_close(f_);
  }
  std::uint64_t push(const float* frame) {
    std::uint64_t seq = 0;
    detail::check(st_frames_push(f_, frame, &seq));
    return seq;
  }
  spectree::ClassAssignment pop(std::uint64_t seq) {
    spectree::ClassAssignment out(records_);
    detail::check(st_frames_pop(f_, seq, out.data()));
    return out;
  }
  void slot(std::uint64_t seq, float** records, std::uint32_t** labels) {
    detail::check(st_frames_slot(f_, seq, records, labels));
  }
  void acquire(std::uint64_t seq, void* stream) { detail::check(st_frames_acquire(f_, seq, stream)); }
  void publish(std::uint64_t seq, void* stream) { detail::check(st_frames_publish(f_, seq, stream)); }
  void wait(std::uint64_t seq, void* stream) { detail::check(st_frames_wait(f_, seq, stream)); }
  void close() {
    st_frames* f = f_;
    f_ = nullptr;
    if (f) detail::check(st_frames_close(f));
  }

 private:
  detail::TreeHandle tree_;  // outlives the stream (declared first, destroyed last)
  std::uint64_t records_;
  st_frames* f_ = nullptr;
};

}  // namespace spectree_b200

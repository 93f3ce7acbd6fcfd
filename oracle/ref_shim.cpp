// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C-ABI shim over the *unmodified* reference `spectree` core, compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/.  It lets
// the Python tests, smoke() and bench.py's CPU-baseline / reference arm call
// the reference's own generators and evaluators:
//
//   generate_synthetic_tree / generate_synthetic_dataset  (synthetic.cpp:82-182)
//   eval_serial                                           (eval_serial.cpp:33-41)
//   eval_data_parallel                                    (eval_data_parallel.cpp:35-88)
//   eval_speculative / eval_speculative_basic + stats     (eval_speculative.cpp:207-273)
//   traversal_depths                                      (eval_serial.cpp:77-93)
//   dataset_checksum / tile_dataset                       (dataset.cpp:35-93)
//   load_tree_json / tree_to_json                         (io.cpp:156-263)
//   validate                                              (tree.cpp:138-189)
//   simulate_data_parallel / simulate_speculative         (warp_sim.cpp:30-274)
//
// Errors are caught and returned as the CLI's exit-code taxonomy
// (main.cpp:703-712): 2 = ArgumentError family, 3 = other spectree::Error.

#include <spectree/dataset.hpp>
#include <spectree/errors.hpp>
#include <spectree/eval_data_parallel.hpp>
#include <spectree/eval_serial.hpp>
#include <spectree/eval_speculative.hpp>
#include <spectree/io.hpp>
#include <spectree/synthetic.hpp>
#include <spectree/tree.hpp>
#include <spectree/warp_sim.hpp>

#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

using namespace spectree;

static_assert(sizeof(EncodedNode) == 16, "EncodedNode must stay 16 bytes");

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_error.clear();
    return 0;
  } catch (const ArgumentError& e) {
    g_error = e.what();
    return 2;
  } catch (const Error& e) {
    g_error = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 4;
  }
}

struct RefTree {
  EncodedTree tree;
};
struct RefData {
  Dataset data;
};

EncodedTree make_tree(const void* nodes, std::uint32_t n) {
  std::vector<EncodedNode> v(n);
  if (n) std::memcpy(v.data(), nodes, sizeof(EncodedNode) * n);
  return EncodedTree(std::move(v));
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_error.c_str(); }

// --- canonical inputs -----------------------------------------------------

// Writes at most `cap` nodes; *n_out receives the true node count.
int ref_gen_tree(std::uint32_t depth, std::uint32_t leaves, std::uint32_t arity,
                 std::uint32_t classes, std::uint64_t seed, void* out,
                 std::uint32_t cap, std::uint32_t* n_out) {
  return guarded([&] {
    EncodedTree t = generate_synthetic_tree(depth, leaves, arity, classes, seed);
    *n_out = t.size();
    if (out && cap >= t.size())
      std::memcpy(out, t.nodes().data(), sizeof(EncodedNode) * t.size());
  });
}

int ref_gen_dataset(std::uint64_t count, std::uint32_t arity, std::uint64_t seed,
                    int gaussian, float* out) {
  return guarded([&] {
    Dataset d = generate_synthetic_dataset(
        count, arity, seed, gaussian ? Distribution::gaussian : Distribution::uniform);
    std::memcpy(out, d.values().data(), d.values().size_bytes());
  });
}

std::uint64_t ref_dataset_checksum(const float* x, std::uint64_t m, std::uint32_t a) {
  Dataset d(a, std::vector<float>(x, x + m * a));
  return dataset_checksum(d);
}

// --- handles (construction kept outside timed regions) --------------------

int ref_tree_create(const void* nodes, std::uint32_t n, void** out) {
  return guarded([&] { *out = new RefTree{make_tree(nodes, n)}; });
}
void ref_tree_destroy(void* t) { delete static_cast<RefTree*>(t); }
std::uint32_t ref_tree_depth(void* t) { return static_cast<RefTree*>(t)->tree.depth(); }
std::uint32_t ref_tree_max_attribute(void* t) {
  return static_cast<RefTree*>(t)->tree.max_attribute();
}
std::uint32_t ref_tree_leaf_count(void* t) {
  return static_cast<RefTree*>(t)->tree.leaf_count();
}
// Number of validate() findings (tree.cpp:138-189); 0 = well formed.
std::uint32_t ref_tree_validate(void* t) {
  return static_cast<std::uint32_t>(validate(static_cast<RefTree*>(t)->tree).size());
}

int ref_data_create(const float* x, std::uint64_t m, std::uint32_t a, void** out) {
  return guarded([&] {
    *out = new RefData{Dataset(a, std::vector<float>(x, x + m * a))};
  });
}
void ref_data_destroy(void* d) { delete static_cast<RefData*>(d); }

// --- evaluators -----------------------------------------------------------

int ref_eval_serial(void* t, void* d, std::uint32_t* out) {
  return guarded([&] {
    ClassAssignment r = eval_serial(static_cast<RefTree*>(t)->tree,
                                    static_cast<RefData*>(d)->data);
    std::memcpy(out, r.data(), r.size() * 4);
  });
}

int ref_eval_data_parallel(void* t, void* d, std::uint32_t workers,
                           std::uint32_t chunk, int exact_fit,
                           std::uint32_t os_threads, std::uint32_t* out) {
  return guarded([&] {
    DataParallelConfig c;
    c.workers = workers;
    c.chunk = chunk;
    c.exact_fit = exact_fit != 0;
    c.os_threads = os_threads;
    ClassAssignment r = eval_data_parallel(static_cast<RefTree*>(t)->tree,
                                           static_cast<RefData*>(d)->data, c);
    std::memcpy(out, r.data(), r.size() * 4);
  });
}

// basic != 0 selects eval_speculative_basic (all lanes).  iters / steps may be
// null; when given they receive SpeculativeStats per record.
int ref_eval_speculative(void* t, void* d, std::uint32_t group_lanes,
                         std::uint32_t groups, std::uint32_t records_per_group,
                         std::uint32_t reductions, int compound, int basic,
                         std::uint32_t os_threads, std::uint32_t* out,
                         std::uint32_t* iters, std::uint32_t* steps,
                         std::uint64_t* barriers) {
  return guarded([&] {
    SpeculativeConfig c;
    c.group_lanes = group_lanes;
    c.groups = groups;
    c.records_per_group = records_per_group;
    c.reductions_per_iteration = reductions;
    c.mode = compound ? ReductionMode::compound_in_place
                      : ReductionMode::barrier_separated;
    c.os_threads = os_threads;
    SpeculativeStats stats;
    const EncodedTree& tree = static_cast<RefTree*>(t)->tree;
    const Dataset& data = static_cast<RefData*>(d)->data;
    ClassAssignment r = basic ? eval_speculative_basic(tree, data, c, &stats)
                              : eval_speculative(tree, data, c, &stats);
    std::memcpy(out, r.data(), r.size() * 4);
    if (iters) std::memcpy(iters, stats.iterations.data(), r.size() * 4);
    if (steps) std::memcpy(steps, stats.doubling_steps.data(), r.size() * 4);
    if (barriers) *barriers = stats.barriers;
  });
}

int ref_traversal_depths(void* t, void* d, std::uint32_t* out) {
  return guarded([&] {
    std::vector<std::uint32_t> r = traversal_depths(static_cast<RefTree*>(t)->tree,
                                                    static_cast<RefData*>(d)->data);
    std::memcpy(out, r.data(), r.size() * 4);
  });
}

// --- lockstep warp model (warp_sim.cpp) ------------------------------------
// out[6] = {divergent_branches, serialized_passes, barriers, node_evals,
//           reduction_iterations, lane_idle_slots} (warp_sim.hpp:37-44)
static void put_metrics(const ExecMetrics& m, std::uint64_t* out) {
  out[0] = m.divergent_branches;
  out[1] = m.serialized_passes;
  out[2] = m.barriers;
  out[3] = m.node_evals;
  out[4] = m.reduction_iterations;
  out[5] = m.lane_idle_slots;
}

int ref_simulate_data_parallel(void* t, void* d, std::uint32_t warp_width, int half_warp,
                               std::uint32_t workers, std::uint32_t chunk, std::uint64_t* out) {
  return guarded([&] {
    WarpConfig w;
    w.warp_width = warp_width;
    w.half_warp = half_warp != 0;
    DataParallelConfig c;
    c.workers = workers;
    c.chunk = chunk;
    put_metrics(simulate_data_parallel(static_cast<RefTree*>(t)->tree, static_cast<RefData*>(d)->data, w, c),
                out);
  });
}

int ref_simulate_speculative(void* t, void* d, std::uint32_t warp_width, int half_warp,
                             std::uint32_t group_lanes, std::uint32_t groups,
                             std::uint32_t records_per_group, std::uint32_t reductions, int basic,
                             std::uint64_t* out) {
  return guarded([&] {
    WarpConfig w;
    w.warp_width = warp_width;
    w.half_warp = half_warp != 0;
    SpeculativeConfig c;
    c.group_lanes = group_lanes;
    c.groups = groups;
    c.records_per_group = records_per_group;
    c.reductions_per_iteration = reductions;
    put_metrics(simulate_speculative(static_cast<RefTree*>(t)->tree, static_cast<RefData*>(d)->data, w, c,
                                     basic ? SpeculativeVariant::all_lanes : SpeculativeVariant::mapped_lanes),
                out);
  });
}

// --- tree JSON (io.cpp) ---------------------------------------------------

// Parses JSON text; *n_out = node count; nodes copied when cap suffices.
int ref_load_tree_json(const char* text, void* out, std::uint32_t cap,
                       std::uint32_t* n_out) {
  return guarded([&] {
    std::istringstream in(text);
    EncodedTree t = load_tree_json(in, "<memory>");
    *n_out = t.size();
    if (out && cap >= t.size())
      std::memcpy(out, t.nodes().data(), sizeof(EncodedNode) * t.size());
  });
}

// Returns the byte length of tree_to_json; copies when cap suffices.
std::uint64_t ref_tree_to_json(const void* nodes, std::uint32_t n, char* out,
                               std::uint64_t cap) {
  std::string s = tree_to_json(make_tree(nodes, n));
  if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
  return s.size();
}

}  // extern "C"

// TEST INFRASTRUCTURE ONLY.
//
// Runs the reference's own acceptance corpus through the C++ drop-in
// (include/spectree_b200.hpp) on the GPU and checks it against the
// reference's own evaluators, compiled unchanged from /root/reference:
//
//   criterion 1 (acceptance.cpp:71-168): every full tree shape up to 8 leaves
//     on grid records + 1000 fuzz trees (depth 1-20, 1000 records, arity 1-8,
//     uniform/gaussian): GPU data-parallel, speculative (mapped, k = 1..3) and
//     speculative-basic vs eval_oracle_recursive -- zero mismatches;
//   criterion 2 (acceptance.cpp:173-211): per-record doubling counters of the
//     GPU speculative kernel vs the law ceil(log2 depth) (and the paired
//     k = 2 law), on the reference's own workload (39 internal nodes: the
//     CTA-scope exact kernel) and 40 trees that fit one warp group (shfl);
//   traversal depths: spectree_b200::traversal_depths (the data kernel's
//     depth output) vs the reference traversal_depths on the same corpus;
//   sharded: eval_data_parallel through GpuConfig.devices (every GPU of the
//     box, or device 0 twice on a one-GPU box) vs the oracle;
//   error behaviour: ArgumentError before any work, with the reference text;
//   frames: spectree_b200::FrameStream (the resident frame stream) per frame
//     vs the reference eval_serial.
//
// Built by oracle/Makefile into oracle/_ref/gpu_acceptance (needs the GPU
// library); tests/test_gpu.py runs it.  Prints one PASS/FAIL line per check,
// exit status = number of failures.
#include <spectree/dataset.hpp>
#include <spectree/errors.hpp>
#include <spectree/eval_data_parallel.hpp>
#include <spectree/eval_serial.hpp>
#include <spectree/eval_speculative.hpp>
#include <spectree/synthetic.hpp>
#include <spectree/tree.hpp>

#include "test_support.hpp"  // the reference's fixtures (tests/unit)

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <string>

#include "spectree_b200.hpp"

using namespace spectree;

namespace {

int failures = 0;

void report(bool ok, const std::string& name, const std::string& detail) {
  std::printf("%s %s: %s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.c_str());
  if (!ok) ++failures;
}

std::uint32_t ceil_log2(std::uint32_t d) {
  std::uint32_t s = 0, reach = 1;
  while (reach < d) {
    reach *= 2;
    ++s;
  }
  return s;
}

std::uint32_t div_ceil(std::uint32_t a, std::uint32_t b) { return (a + b - 1) / b; }

std::string check_all(const EncodedTree& tree, const LinkedNode& root, const Dataset& data,
                      std::uint32_t k, std::uint64_t salt) {
  const ClassAssignment expected = eval_oracle_recursive(root, data);
  DataParallelConfig dp;
  dp.workers = 3 + salt % 5;
  dp.chunk = std::max(1u, div_ceil(static_cast<std::uint32_t>(data.count()), dp.workers));
  if (spectree_b200::eval_data_parallel(tree, data, dp) != expected) return "gpu data-parallel";
  if (spectree_b200::traversal_depths(tree, data) != traversal_depths(tree, data))
    return "gpu traversal depths";
  {
    spectree_b200::GpuConfig sharded;
    int n = 1;
    st_device_count(&n);
    for (int d = 0; d < std::max(2, n); ++d) sharded.devices.push_back(d % n);
    if (spectree_b200::eval_data_parallel(tree, data, dp, sharded) != expected)
      return "gpu data-parallel sharded over " + std::to_string(sharded.devices.size()) + " devices";
  }
  SpeculativeConfig basic;
  basic.group_lanes = tree.size();
  basic.records_per_group = 1 + salt % 4;
  basic.groups = std::max(1u, div_ceil(static_cast<std::uint32_t>(data.count()),
                                       basic.records_per_group));
  basic.reductions_per_iteration = 1;
  if (spectree_b200::eval_speculative_basic(tree, data, basic) != expected)
    return "gpu speculative-basic";
  SpeculativeConfig mapped = basic;
  mapped.group_lanes = std::max(1u, (tree.size() - 1) / 2);
  mapped.reductions_per_iteration = k;
  if (spectree_b200::eval_speculative(tree, data, mapped) != expected) return "gpu speculative";
  spectree_b200::GpuConfig g16;
  g16.geom.group_lanes = 16;  // windowed geometry regardless of tree size
  if (spectree_b200::eval_speculative(tree, data, mapped, nullptr, g16) != expected)
    return "gpu speculative (G=16 windows)";
  return {};
}

void criterion1() {
  const auto start = std::chrono::steady_clock::now();
  std::uint64_t shapes = 0, records = 0;
  for (std::uint32_t leaves = 1; leaves <= 8; ++leaves) {
    for (auto& shape : testsupport::all_shapes(leaves)) {
      const std::uint32_t internal = testsupport::assign_labels(*shape);
      const Dataset grid = testsupport::grid_records(internal);
      const EncodedTree tree = encode_breadth_first(*shape);
      const std::string err = check_all(tree, *shape, grid, 2, shapes);
      if (!err.empty()) {
        report(false, "criterion1", err + " on a shape with " + std::to_string(leaves) + " leaves");
        return;
      }
      ++shapes;
      records += grid.count();
    }
  }
  for (std::uint64_t seed = 1; seed <= 1000; ++seed) {
    const std::uint32_t depth = 1 + seed % 20;
    const std::uint32_t lo = depth + 1;
    const std::uint32_t cap = depth >= 10 ? 1024u : (1u << depth);
    const std::uint32_t hi = std::min(cap, lo + 19);
    const std::uint32_t leaves = lo + static_cast<std::uint32_t>((seed * 7) % (hi - lo + 1));
    const std::uint32_t arity = 1 + static_cast<std::uint32_t>((seed * 3) % 8);
    const std::uint32_t classes = 2 + static_cast<std::uint32_t>(seed % 9);
    const EncodedTree tree = generate_synthetic_tree(depth, leaves, arity, classes, seed);
    const Dataset data = generate_synthetic_dataset(
        1000, arity, seed + 5000, seed % 2 ? Distribution::uniform : Distribution::gaussian);
    const auto linked = decode(tree);
    const std::string err = check_all(tree, *linked, data, 1 + seed % 3, seed);
    if (!err.empty()) {
      report(false, "criterion1", err + " at fuzz seed " + std::to_string(seed));
      return;
    }
    records += data.count();
  }
  const double s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
  report(true, "criterion1",
         std::to_string(shapes) + " exhaustive shapes + 1000 fuzz trees, " +
             std::to_string(records) + " records, 0 mismatches on the GPU (" +
             std::to_string(s).substr(0, 5) + " s)");
}

void criterion2() {
  std::uint64_t trees = 0, recs = 0;
  // seed 0 is the reference's own criterion-2 workload (acceptance.cpp:174-176,
  // 39 internal nodes); seeds 1..40 add trees that fit one warp group
  for (std::uint64_t seed = 0; seed <= 40; ++seed) {
    const EncodedTree tree = seed == 0 ? generate_synthetic_tree(20, 40, 8, 5, 97)
                                       : generate_synthetic_tree(12, 20 + seed % 13, 8, 5, 97 + seed);
    const Dataset data = seed == 0 ? generate_synthetic_dataset(10000, 8, 13, Distribution::uniform)
                                   : generate_synthetic_dataset(10000, 8, 13 + seed, Distribution::uniform);
    const auto depths = traversal_depths(tree, data);
    SpeculativeConfig config;
    config.group_lanes = (tree.size() - 1) / 2;
    config.records_per_group = 16;
    config.groups = div_ceil(10000, 16);
    config.reductions_per_iteration = 1;
    SpeculativeStats single;
    spectree_b200::eval_speculative(tree, data, config, &single);
    config.reductions_per_iteration = 2;
    SpeculativeStats paired;
    spectree_b200::eval_speculative(tree, data, config, &paired);
    for (std::size_t r = 0; r < data.count(); ++r) {
      const std::uint32_t want = ceil_log2(depths[r]);
      if (single.doubling_steps[r] != want || single.iterations[r] != want ||
          paired.iterations[r] != div_ceil(want, 2)) {
        report(false, "criterion2", "record " + std::to_string(r) + " of seed " +
                                        std::to_string(seed) + " breaks the doubling law");
        return;
      }
    }
    ++trees;
    recs += data.count();
  }
  report(true, "criterion2",
         std::to_string(recs) + " records over " + std::to_string(trees) +
             " trees: single doublings = ceil(log2 depth), paired iterations = ceil(/2)");
}

void errors() {
  auto linked = make_split(5, 0.5f, make_leaf(1), make_leaf(2));
  EncodedTree tree = encode_breadth_first(*linked);
  Dataset narrow(2, {0.1f, 0.2f});
  std::string ref_msg, gpu_msg;
  try {
    eval_serial(tree, narrow);
  } catch (const ArgumentError& e) {
    ref_msg = e.what();
  }
  try {
    DataParallelConfig dp;
    spectree_b200::eval_data_parallel(tree, narrow, dp);
  } catch (const ArgumentError& e) {
    gpu_msg = e.what();
  }
  report(!ref_msg.empty() && ref_msg == gpu_msg, "errors",
         "attribute range -> ArgumentError \"" + gpu_msg + "\"");
  DataParallelConfig bad;
  bad.workers = 0;
  bool threw = false;
  try {
    spectree_b200::eval_data_parallel(tree, Dataset(6, {0, 0, 0, 0, 0, 0}), bad);
  } catch (const ArgumentError&) {
    threw = true;
  }
  report(threw, "geometry", "workers == 0 -> ArgumentError before any work");
  Dataset empty(6);
  DataParallelConfig one;
  report(spectree_b200::eval_data_parallel(tree, empty, one).empty(), "empty",
         "empty dataset -> empty assignment");
  std::string ref_d, gpu_d;
  try {
    mean_traversal_depth(tree, empty);
  } catch (const ArgumentError& e) {
    ref_d = e.what();
  }
  try {
    spectree_b200::mean_traversal_depth(tree, empty);
  } catch (const ArgumentError& e) {
    gpu_d = e.what();
  }
  report(!ref_d.empty() && ref_d == gpu_d, "empty-depth",
         "mean traversal depth of an empty dataset -> ArgumentError \"" + gpu_d + "\"");
}

// The resident frame stream through the C++ wrapper: a C3-shaped tree
// (depth 12, 2048 leaves, 8 attributes), 7 frames of 16384 records through a
// 3-slot ring, each frame's labels vs the reference eval_serial.
void frames() {
  const EncodedTree tree = generate_synthetic_tree(12, 2048, 8, 8, 301);
  bool ok = true;
  std::string detail = "7 frames x 16384 records, ring 3: labels == eval_serial";
  try {
    spectree_b200::FrameStream fs(tree, 16384, 8, 3, {}, 20000);
    std::vector<Dataset> frames_;
    std::vector<std::uint64_t> seqs;
    for (int k = 0; k < 7; ++k) frames_.push_back(generate_synthetic_dataset(16384, 8, 4000 + k, k % 2 == 1 ? Distribution::gaussian : Distribution::uniform));
    std::size_t popped = 0;
    for (int k = 0; k < 7; ++k) {
      if (seqs.size() - popped == 3) {
        ok = ok && fs.pop(seqs[popped]) == eval_serial(tree, frames_[popped]);
        ++popped;
      }
      seqs.push_back(fs.push(frames_[k].values().data()));
    }
    for (; popped < seqs.size(); ++popped) ok = ok && fs.pop(seqs[popped]) == eval_serial(tree, frames_[popped]);
    fs.close();
  } catch (const std::exception& e) {
    ok = false;
    detail = e.what();
  }
  report(ok, "frames", detail);
}

}  // namespace

int main() {
  int n = 0;
  st_device_count(&n);
  if (n == 0) {
    std::printf("SKIP no CUDA device\n");
    return 0;
  }
  errors();
  criterion1();
  criterion2();
  frames();
  return failures;
}

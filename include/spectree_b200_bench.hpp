// spectree_b200_bench.hpp -- the reference's verify/bench flow with GPU
// strategies, header-only over the C ABI.
//
// Mirrors /root/reference/proj/core/include/spectree/bench.hpp type for type
// (Strategy, strategy_name / strategy_from_name, TimingStats, summarize,
// StrategyComparison, verify_strategies, BenchConfig, StrategyReport,
// BenchReport, run_bench, report_to_json / report_to_table), adding two
// strategies that run on the GPU through this library:
//
//   gpu-data   Algorithm 1 on the GPU (spectree_b200::eval_data_parallel)
//   gpu-spec   Algorithm 2 on the GPU (spectree_b200::eval_speculative)
//
// Timing windows keep the reference's meaning (bench.hpp:50-56,
// bench.cpp:228-262): for a GPU strategy "outer" is one whole round trip --
// device allocation, records host->device, kernel, labels device->host,
// release -- "inner" is the kernel alone (CUDA events) and "alloc" is the
// device allocation + release; the paper's Table 1 columns.  The CPU
// strategies call the reference's own evaluators unchanged, so this header
// is compiled inside the reference build (it includes <spectree/*.hpp> and
// <json.hpp> exactly like bench.cpp:1-14).
//
// run_kernel / verify_strategies replace bench.cpp:60-76 / :153-166;
// run_bench replaces :168-281; report_to_json keeps schema version 1
// (:301-355) with the GPU names and an extra "gpu" object per GPU strategy
// (h2d_us / d2h_us means).
#pragma once

#include <spectree/bench.hpp>
#include <spectree/dataset.hpp>
#include <spectree/errors.hpp>
#include <spectree/eval_data_parallel.hpp>
#include <spectree/eval_serial.hpp>
#include <spectree/eval_speculative.hpp>
#include <spectree/tree.hpp>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <optional>
#include <span>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include <json.hpp>

#include "spectree_b200.h"
#include "spectree_b200.hpp"

namespace spectree_b200 {

enum class Strategy { serial, data_parallel, speculative, speculative_basic, gpu_data, gpu_spec };

inline const char* strategy_name(Strategy s) {  // bench.cpp:98-110 + GPU names
  switch (s) {
    case Strategy::serial: return "serial";
    case Strategy::data_parallel: return "data";
    case Strategy::speculative: return "spec";
    case Strategy::speculative_basic: return "spec-basic";
    case Strategy::gpu_data: return "gpu-data";
    case Strategy::gpu_spec: return "gpu-spec";
  }
  return "unknown";
}

inline std::optional<Strategy> strategy_from_name(std::string_view name) {  // bench.cpp:112-126
  for (Strategy s : {Strategy::serial, Strategy::data_parallel, Strategy::speculative,
                     Strategy::speculative_basic, Strategy::gpu_data, Strategy::gpu_spec})
    if (name == strategy_name(s)) return s;
  return std::nullopt;
}

inline bool is_gpu(Strategy s) { return s == Strategy::gpu_data || s == Strategy::gpu_spec; }

using spectree::summarize;
using spectree::TimingStats;

struct StrategyComparison {  // bench.hpp:35-44
  Strategy strategy = Strategy::serial;
  std::uint64_t mismatches = 0;
  std::optional<std::uint64_t> first_mismatch;
  std::uint32_t expected = 0;
  std::uint32_t actual = 0;
  [[nodiscard]] bool matches() const noexcept { return mismatches == 0; }
};

namespace detail {

inline spectree::SpeculativeConfig basic_config(const spectree::SpeculativeConfig& c,
                                                const spectree::EncodedTree& tree) {
  spectree::SpeculativeConfig b = c;  // bench.cpp:52-58
  b.group_lanes = tree.size();
  return b;
}

inline StrategyComparison compare(Strategy s, const spectree::ClassAssignment& ref,
                                  const spectree::ClassAssignment& got) {  // bench.cpp:78-94
  StrategyComparison c;
  c.strategy = s;
  for (std::size_t i = 0; i < ref.size(); ++i) {
    if (got[i] != ref[i]) {
      if (c.mismatches == 0) {
        c.first_mismatch = i;
        c.expected = ref[i];
        c.actual = got[i];
      }
      ++c.mismatches;
    }
  }
  return c;
}

inline st_geom gpu_geom(Strategy s, const GpuConfig& gpu) {
  st_geom g = gpu.geom;
  g.algo = s == Strategy::gpu_spec ? ST_ALGO_SPECULATIVE : ST_ALGO_DATA;
  return g;
}

}  // namespace detail

/// bench.cpp:60-76 with the GPU strategies.  GPU strategies validate the
/// reference configs first (same ArgumentError as the CPU strategy), then
/// evaluate on the GPU.
inline spectree::ClassAssignment run_kernel(Strategy s, const spectree::EncodedTree& tree,
                                            const spectree::Dataset& data,
                                            const spectree::DataParallelConfig& dp,
                                            const spectree::SpeculativeConfig& sp,
                                            const GpuConfig& gpu = {}) {
  switch (s) {
    case Strategy::serial: return spectree::eval_serial(tree, data);
    case Strategy::data_parallel: return spectree::eval_data_parallel(tree, data, dp);
    case Strategy::speculative: return spectree::eval_speculative(tree, data, sp);
    case Strategy::speculative_basic:
      return spectree::eval_speculative_basic(tree, data, detail::basic_config(sp, tree));
    case Strategy::gpu_data: return eval_data_parallel(tree, data, dp, gpu);
    case Strategy::gpu_spec: return eval_speculative(tree, data, sp, nullptr, gpu);
  }
  throw spectree::ArgumentError("unknown strategy");
}

inline std::vector<StrategyComparison> verify_strategies(const spectree::EncodedTree& tree,
                                                         const spectree::Dataset& data,
                                                         std::span<const Strategy> strategies,
                                                         const spectree::DataParallelConfig& dp,
                                                         const spectree::SpeculativeConfig& sp,
                                                         const GpuConfig& gpu = {}) {
  const spectree::ClassAssignment ref = spectree::eval_serial(tree, data);
  std::vector<StrategyComparison> out;
  for (Strategy s : strategies) out.push_back(detail::compare(s, ref, run_kernel(s, tree, data, dp, sp, gpu)));
  return out;
}

struct BenchConfig {  // bench.hpp:46-55 (+ GPU geometry)
  std::vector<Strategy> strategies{Strategy::serial};
  std::uint32_t iterations = 500;
  std::uint32_t warmup = 10;
  spectree::DataParallelConfig data_parallel{};
  spectree::SpeculativeConfig speculative{};
  bool keep_samples = false;
  GpuConfig gpu{};
};

struct GpuPhases {  // per-iteration means of the copy windows (GPU strategies)
  double h2d_mean_us = 0;
  double d2h_mean_us = 0;
};

struct StrategyReport {  // bench.hpp:58-78
  Strategy strategy = Strategy::serial;
  TimingStats outer;
  std::optional<TimingStats> inner;
  std::optional<TimingStats> alloc;
  std::optional<GpuPhases> gpu;
  std::vector<double> outer_samples_us;
  std::vector<double> inner_samples_us;
  StrategyComparison verification;
};

struct BenchReport {  // bench.hpp:80-97
  std::string os;
  std::uint32_t hardware_threads = 0;
  std::string device;
  std::uint32_t iterations = 0;
  std::uint32_t warmup = 0;
  double timer_overhead_us = 0;
  spectree::TreeStats tree;
  std::uint64_t records = 0;
  std::uint32_t arity = 0;
  std::uint64_t checksum_before = 0;
  std::uint64_t checksum_after = 0;
  spectree::DataParallelConfig data_parallel;
  spectree::SpeculativeConfig speculative;
  std::vector<StrategyReport> strategies;
  bool all_match = true;
};

namespace detail {

using Clock = std::chrono::steady_clock;
inline double to_us(Clock::duration d) { return std::chrono::duration<double, std::micro>(d).count(); }

inline double timer_overhead() {  // bench.cpp:28-38
  std::vector<double> d(1000);
  for (double& x : d) {
    const auto a = Clock::now();
    const auto b = Clock::now();
    x = to_us(b - a);
  }
  std::nth_element(d.begin(), d.begin() + d.size() / 2, d.end());
  return d[d.size() / 2];
}

}  // namespace detail

/// bench.cpp:168-281 with the GPU strategies.  Geometry is validated before
/// any clock starts, warm-up iterations are excluded, the dataset is
/// checksummed around the runs, every strategy is verified against
/// eval_serial computed outside the timed region.
inline BenchReport run_bench(const spectree::EncodedTree& tree, const spectree::Dataset& data,
                             const BenchConfig& cfg) {
  if (cfg.iterations == 0) throw spectree::ArgumentError("bench iterations must be >= 1");
  if (cfg.strategies.empty()) throw spectree::ArgumentError("bench requires at least one strategy");
  spectree::check_attribute_range(tree, data);
  for (Strategy s : cfg.strategies) {
    switch (s) {
      case Strategy::serial: break;
      case Strategy::data_parallel:
      case Strategy::gpu_data: spectree::validate_data_parallel(cfg.data_parallel, data.count()); break;
      case Strategy::speculative:
      case Strategy::gpu_spec:
        spectree::validate_speculative(cfg.speculative, tree, data.count(), false);
        break;
      case Strategy::speculative_basic:
        spectree::validate_speculative(detail::basic_config(cfg.speculative, tree), tree, data.count(),
                                       true);
        break;
    }
  }
  BenchReport rep;
  rep.os = "linux";
  rep.hardware_threads = std::max(1u, std::thread::hardware_concurrency());
  rep.iterations = cfg.iterations;
  rep.warmup = cfg.warmup;
  rep.tree = spectree::stats(tree);
  rep.records = data.count();
  rep.arity = data.arity();
  rep.data_parallel = cfg.data_parallel;
  rep.speculative = cfg.speculative;
  rep.checksum_before = spectree::dataset_checksum(data);
  const spectree::ClassAssignment ref = spectree::eval_serial(tree, data);
  rep.timer_overhead_us = detail::timer_overhead();

  detail::TreeHandle handle;  // one device tree for every GPU iteration
  for (Strategy s : cfg.strategies) {
    StrategyReport e;
    e.strategy = s;
    std::vector<double> outer, inner, alloc;
    double h2d = 0, d2h = 0;
    spectree::ClassAssignment last;
    const std::uint64_t total = (std::uint64_t)cfg.warmup + cfg.iterations;
    if (is_gpu(s) && !handle) handle = detail::make_handle(tree);
    for (std::uint64_t i = 0; i < total; ++i) {
      const bool timed = i >= cfg.warmup;
      if (is_gpu(s)) {
        spectree::ClassAssignment out(data.count());
        const st_geom g = detail::gpu_geom(s, cfg.gpu);
        st_timing t{};
        if (data.count())
          detail::check(st_eval_timed(handle.get(), data.values().data(), data.count(), data.arity(), 0,
                                      ST_LAYOUT_AOS, &g, out.data(), &t));
        if (timed) {
          outer.push_back(t.outer_us);
          inner.push_back(t.inner_us);
          alloc.push_back(t.alloc_us);
          h2d += t.h2d_us;
          d2h += t.d2h_us;
        }
        last = std::move(out);
        continue;
      }
      if (s == Strategy::serial) {  // in place, outer only (bench.cpp:232-243)
        const auto o0 = detail::Clock::now();
        spectree::ClassAssignment r = spectree::eval_serial(tree, data);
        const auto o1 = detail::Clock::now();
        if (timed) outer.push_back(detail::to_us(o1 - o0));
        last = std::move(r);
        continue;
      }
      // CPU strategies: the reference's staging round trip (bench.cpp:244-262)
      const auto o0 = detail::Clock::now();
      std::vector<float> values;
      std::vector<spectree::EncodedNode> nodes;
      values.reserve(data.values().size());
      nodes.reserve(tree.size());
      const auto a1 = detail::Clock::now();
      values.insert(values.end(), data.values().begin(), data.values().end());
      nodes.assign(tree.nodes().begin(), tree.nodes().end());
      std::optional<spectree::Dataset> staged(std::in_place, data.arity(), std::move(values));
      std::optional<spectree::EncodedTree> staged_tree(std::in_place, std::move(nodes));
      const auto i0 = detail::Clock::now();
      spectree::ClassAssignment r =
          run_kernel(s, *staged_tree, *staged, cfg.data_parallel, cfg.speculative, cfg.gpu);
      const auto i1 = detail::Clock::now();
      last = r;
      const auto f0 = detail::Clock::now();
      staged.reset();
      staged_tree.reset();
      const auto f1 = detail::Clock::now();
      if (timed) {
        outer.push_back(detail::to_us(f1 - o0));
        inner.push_back(detail::to_us(i1 - i0));
        alloc.push_back(detail::to_us(a1 - o0) + detail::to_us(f1 - f0));
      }
    }
    e.outer = summarize(outer);
    if (!inner.empty()) {
      e.inner = summarize(inner);
      e.alloc = summarize(alloc);
    }
    if (is_gpu(s)) e.gpu = GpuPhases{h2d / cfg.iterations, d2h / cfg.iterations};
    if (cfg.keep_samples) {
      e.outer_samples_us = outer;
      e.inner_samples_us = inner;
    }
    e.verification = detail::compare(s, ref, last);
    rep.all_match = rep.all_match && e.verification.matches();
    rep.strategies.push_back(std::move(e));
  }
  rep.checksum_after = spectree::dataset_checksum(data);
  if (rep.checksum_after != rep.checksum_before)
    throw spectree::Error("dataset checksum changed during benchmarking");
  return rep;
}

/// Schema version 1 of bench.cpp:301-355, GPU strategies included.
inline std::string report_to_json(const BenchReport& r) {
  using nlohmann::json;
  auto st = [](const TimingStats& s) {
    return json{{"mean_us", s.mean_us}, {"min_us", s.min_us}, {"max_us", s.max_us},
                {"stddev_us", s.stddev_us}, {"iterations", s.iterations}};
  };
  auto hex64 = [](std::uint64_t v) {
    char b[19];
    std::snprintf(b, sizeof b, "0x%016llx", static_cast<unsigned long long>(v));
    return std::string(b);
  };
  json doc;
  doc["version"] = 1;
  doc["machine"] = {{"os", r.os}, {"hardware_threads", r.hardware_threads}, {"timer", "steady_clock"}};
  doc["config"] = {
      {"iterations", r.iterations},
      {"warmup", r.warmup},
      {"tree", {{"nodes", r.tree.nodes}, {"leaves", r.tree.leaves}, {"depth", r.tree.depth}}},
      {"dataset", {{"records", r.records}, {"arity", r.arity}}},
      {"data_parallel",
       {{"workers", r.data_parallel.workers}, {"chunk", r.data_parallel.chunk},
        {"exact_fit", r.data_parallel.exact_fit}}},
      {"speculative",
       {{"group_lanes", r.speculative.group_lanes}, {"groups", r.speculative.groups},
        {"records_per_group", r.speculative.records_per_group},
        {"reductions_per_iteration", r.speculative.reductions_per_iteration},
        {"mode", r.speculative.mode == spectree::ReductionMode::barrier_separated ? "barrier-separated"
                                                                                  : "compound-in-place"}}},
      {"metrics_collected", false}};
  doc["timer_overhead_us"] = r.timer_overhead_us;
  doc["dataset_checksum_before"] = hex64(r.checksum_before);
  doc["dataset_checksum_after"] = hex64(r.checksum_after);
  json arr = json::array();
  for (const StrategyReport& e : r.strategies) {
    json it;
    it["name"] = strategy_name(e.strategy);
    it["outer_us"] = st(e.outer);
    it["inner_us"] = e.inner ? st(*e.inner) : json();
    it["alloc_us"] = e.alloc ? st(*e.alloc) : json();
    it["metrics"] = json();
    it["verification"] = {{"matches_serial", e.verification.matches()},
                          {"mismatches", e.verification.mismatches}};
    if (e.gpu) it["gpu"] = {{"h2d_mean_us", e.gpu->h2d_mean_us}, {"d2h_mean_us", e.gpu->d2h_mean_us}};
    if (!e.outer_samples_us.empty())
      it["samples"] = {{"outer_us", e.outer_samples_us}, {"inner_us", e.inner_samples_us}};
    arr.push_back(std::move(it));
  }
  doc["strategies"] = std::move(arr);
  doc["verification"] = {{"reference", "serial"}, {"all_match", r.all_match}};
  return doc.dump(2) + "\n";
}

/// Fixed-width table, one row per strategy (bench.cpp report_to_table shape).
inline std::string report_to_table(const BenchReport& r) {
  auto f3 = [](double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.3f", v);
    return std::string(b);
  };
  auto cell = [](std::string s, std::size_t w) {
    while (s.size() < w) s += ' ';
    return s;
  };
  std::string out = cell("strategy", 12) + cell("outer mean", 14) + cell("outer min", 14) +
                    cell("inner mean", 14) + cell("inner min", 14) + cell("alloc mean", 14) +
                    cell("h2d mean", 12) + cell("d2h mean", 12) + "match\n";
  for (const StrategyReport& e : r.strategies) {
    out += cell(strategy_name(e.strategy), 12) + cell(f3(e.outer.mean_us), 14) + cell(f3(e.outer.min_us), 14) +
           cell(e.inner ? f3(e.inner->mean_us) : "n/a", 14) + cell(e.inner ? f3(e.inner->min_us) : "n/a", 14) +
           cell(e.alloc ? f3(e.alloc->mean_us) : "n/a", 14) +
           cell(e.gpu ? f3(e.gpu->h2d_mean_us) : "n/a", 12) + cell(e.gpu ? f3(e.gpu->d2h_mean_us) : "n/a", 12) +
           (e.verification.matches() ? "yes" : "NO") + "\n";
  }
  return out;
}

}  // namespace spectree_b200

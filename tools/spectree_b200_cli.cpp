// spectree_b200_cli -- the reference CLI's verify / bench subcommands
// (tools/main.cpp:278-420) with the GPU strategy names added,
// plus gen / classify for the binary record format (§8f row 3).
//
//   verify   --tree T.json --data D.(csv|strec) [--strategy S]... [geometry]
//   bench    --tree T.json --data D.(csv|strec) [--strategy S]... [geometry]
//            [--iterations N] [--warmup W] [--format table|json] [--out P]
//   gen      --depth D --leaves L --arity A --classes C --seed S --records M
//            --data-seed S2 --out-tree T.json --out-data D.strec [--soa]
//   classify --tree T.json --data D.strec --out L.stlab [--width 1|4]
//            [--strategy gpu-data|gpu-spec]      (streams the file through the GPU)
//
// Strategies: serial, data, spec, spec-basic (the reference's CPU
// evaluators, unchanged) and gpu-data, gpu-spec (this library).  Geometry
// flags and their defaults are the reference's (main.cpp:60-123).  Exit
// codes are the reference's (main.cpp:37-40, 703-712): 0 ok, 1 mismatch,
// 2 ArgumentError / usage, 3 any other Error.
//
// Built by oracle/Makefile (target `cli`) against the reference sources, like
// the reference's own tools/ target.
#include <spectree/io.hpp>
#include <spectree/synthetic.hpp>

#include <fstream>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "spectree_b200_bench.hpp"

namespace {

using spectree::ArgumentError;

struct Args {
  std::string cmd;
  std::map<std::string, std::string> opt;
  std::vector<std::string> strategies;
  std::vector<std::string> flags;
  std::string get(const std::string& k, const std::string& d = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? d : it->second;
  }
  std::uint64_t num(const std::string& k, std::uint64_t d) const {
    auto it = opt.find(k);
    if (it == opt.end()) return d;
    try {
      return std::stoull(it->second);
    } catch (...) {
      throw ArgumentError("option --" + k + " expects a number, got '" + it->second + "'");
    }
  }
  bool flag(const std::string& f) const {
    for (auto& x : flags)
      if (x == f) return true;
    return false;
  }
  std::string need(const std::string& k) const {
    auto it = opt.find(k);
    if (it == opt.end()) throw ArgumentError("--" + k + " is required");
    return it->second;
  }
};

Args parse(int argc, char** argv) {
  if (argc < 2) throw ArgumentError("usage: spectree_b200_cli verify|bench|gen|classify [options]");
  Args a;
  a.cmd = argv[1];
  static const char* kFlags[] = {"soa", "compound", "verbose"};
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) != 0) throw ArgumentError("unexpected argument '" + s + "'");
    s = s.substr(2);
    bool is_flag = false;
    for (const char* f : kFlags) is_flag = is_flag || s == f;
    if (is_flag) {
      a.flags.push_back(s);
      continue;
    }
    if (i + 1 >= argc) throw ArgumentError("--" + s + " expects a value");
    const std::string v = argv[++i];
    if (s == "strategy") a.strategies.push_back(v);
    else a.opt[s] = v;
  }
  return a;
}

bool ends_with(const std::string& s, const std::string& t) {
  return s.size() >= t.size() && s.compare(s.size() - t.size(), t.size(), t) == 0;
}

spectree::Dataset load_data(const std::string& path) {
  if (ends_with(path, ".csv")) return spectree::load_dataset_csv(path);
  st_dataset_info in{};
  spectree_b200::detail::check(st_dataset_info_read(path.c_str(), &in));
  std::vector<float> v(in.count * in.arity);
  spectree_b200::detail::check(st_dataset_load(path.c_str(), 0, in.count, v.data(), 0));
  return spectree::Dataset(in.arity, std::move(v));
}

// main.cpp:89-123
spectree::DataParallelConfig resolve_data(const Args& a, std::size_t records) {
  spectree::DataParallelConfig c;
  c.workers = (std::uint32_t)a.num("workers", 0);
  if (c.workers == 0) c.workers = std::max(1u, std::thread::hardware_concurrency());
  c.chunk = (std::uint32_t)a.num("chunk", 0);
  if (c.chunk == 0) c.chunk = (std::uint32_t)std::max<std::size_t>(1, (records + c.workers - 1) / c.workers);
  return c;
}

spectree::SpeculativeConfig resolve_spec(const Args& a, const spectree::EncodedTree& t, std::size_t records) {
  spectree::SpeculativeConfig c;
  c.group_lanes = (std::uint32_t)a.num("group-lanes", 0);
  if (c.group_lanes == 0) c.group_lanes = std::max(1u, (t.size() - 1) / 2);
  c.records_per_group = (std::uint32_t)a.num("records-per-group", 32);
  c.groups = (std::uint32_t)a.num("groups", 0);
  if (c.groups == 0)
    c.groups = (std::uint32_t)std::max<std::size_t>(1, (records + c.records_per_group - 1) / c.records_per_group);
  c.reductions_per_iteration = (std::uint32_t)a.num("reductions-per-iter", 2);
  c.mode = a.flag("compound") ? spectree::ReductionMode::compound_in_place
                              : spectree::ReductionMode::barrier_separated;
  return c;
}

std::vector<spectree_b200::Strategy> strategies(const Args& a, std::vector<spectree_b200::Strategy> dflt) {
  if (a.strategies.empty()) return dflt;
  std::vector<spectree_b200::Strategy> out;
  for (auto& n : a.strategies) {
    auto s = spectree_b200::strategy_from_name(n);
    if (!s) throw ArgumentError("unknown strategy '" + n + "'");
    out.push_back(*s);
  }
  return out;
}

using S = spectree_b200::Strategy;

int cmd_verify(const Args& a) {  // main.cpp:278-334
  const auto tree = spectree::load_tree_json(a.need("tree"));
  const auto data = load_data(a.need("data"));
  const auto ss = strategies(a, {S::serial, S::data_parallel, S::speculative, S::speculative_basic,
                                 S::gpu_data, S::gpu_spec});
  const auto dp = resolve_data(a, data.count());
  const auto sp = resolve_spec(a, tree, data.count());
  bool ok = true;
  for (const auto& c : spectree_b200::verify_strategies(tree, data, ss, dp, sp)) {
    if (c.matches()) {
      std::cout << spectree_b200::strategy_name(c.strategy) << ": OK (" << data.count() << " records)\n";
    } else {
      ok = false;
      std::cout << spectree_b200::strategy_name(c.strategy) << ": MISMATCH at record " << *c.first_mismatch
                << ": expected " << c.expected << ", got " << c.actual << " (" << c.mismatches << " total)\n";
    }
  }
  return ok ? 0 : 1;
}

int cmd_bench(const Args& a) {
  const auto tree = spectree::load_tree_json(a.need("tree"));
  const auto data = load_data(a.need("data"));
  spectree_b200::BenchConfig cfg;
  cfg.strategies = strategies(a, {S::serial, S::data_parallel, S::speculative, S::gpu_data, S::gpu_spec});
  cfg.iterations = (std::uint32_t)a.num("iterations", 500);
  cfg.warmup = (std::uint32_t)a.num("warmup", 10);
  cfg.data_parallel = resolve_data(a, data.count());
  cfg.speculative = resolve_spec(a, tree, data.count());
  cfg.keep_samples = a.flag("verbose");
  const auto rep = spectree_b200::run_bench(tree, data, cfg);
  const std::string fmt = a.get("format", "table");
  std::string text;
  if (fmt == "json") text = spectree_b200::report_to_json(rep);
  else if (fmt == "table") text = spectree_b200::report_to_table(rep);
  else throw ArgumentError("unknown format '" + fmt + "'");
  if (a.opt.count("out")) {
    std::ofstream o(a.get("out"));
    if (!o) throw spectree::IoError("cannot open " + a.get("out") + " for writing");
    o << text;
  } else {
    std::cout << text;
  }
  return rep.all_match ? 0 : 1;
}

int cmd_gen(const Args& a) {
  const auto tree = spectree::generate_synthetic_tree(
      (std::uint32_t)a.num("depth", 11), (std::uint32_t)a.num("leaves", 16), (std::uint32_t)a.num("arity", 19),
      (std::uint32_t)a.num("classes", 7), a.num("seed", 1));
  const auto data = spectree::generate_synthetic_dataset(a.num("records", 16384),
                                                          (std::uint32_t)a.num("arity", 19), a.num("data-seed", 2));
  spectree::save_tree_json(tree, a.need("out-tree"));
  const bool soa = a.flag("soa");
  std::vector<float> v(data.values().begin(), data.values().end());
  if (soa) {
    const std::size_t m = data.count(), ar = data.arity();
    std::vector<float> t(v.size());
    for (std::size_t r = 0; r < m; ++r)
      for (std::size_t k = 0; k < ar; ++k) t[k * m + r] = v[r * ar + k];
    v.swap(t);
  }
  spectree_b200::detail::check(st_dataset_save(a.need("out-data").c_str(), v.data(), data.count(), data.arity(),
                                               soa ? ST_LAYOUT_SOA : ST_LAYOUT_AOS, 1));
  return 0;
}

int cmd_classify(const Args& a) {
  const auto tree = spectree::load_tree_json(a.need("tree"));
  const auto ss = strategies(a, {S::gpu_data});
  if (ss.size() != 1 || !spectree_b200::is_gpu(ss[0])) throw ArgumentError("classify takes one GPU strategy");
  spectree_b200::detail::TreeHandle h = spectree_b200::detail::make_handle(tree);
  st_geom g{};
  g.algo = ss[0] == S::gpu_spec ? ST_ALGO_SPECULATIVE : ST_ALGO_DATA;
  std::uint64_t n = 0;
  const auto t0 = std::chrono::steady_clock::now();
  spectree_b200::detail::check(st_eval_file(h.get(), a.need("data").c_str(), &g, a.need("out").c_str(),
                                            (std::uint32_t)a.num("width", 4), &n));
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::cout << "classified " << n << " records in " << s << " s (" << (s > 0 ? n / s : 0.0) << " records/s)\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "verify") return cmd_verify(a);
    if (a.cmd == "bench") return cmd_bench(a);
    if (a.cmd == "gen") return cmd_gen(a);
    if (a.cmd == "classify") return cmd_classify(a);
    throw ArgumentError("unknown subcommand '" + a.cmd + "'");
  } catch (const spectree::ArgumentError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const spectree::Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "unexpected error: " << e.what() << "\n";
    return 3;
  }
}

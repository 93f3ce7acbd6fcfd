// Input-side API of the boundary (reference layer L1, synthetic.hpp:18-30,
// dataset.hpp:27-32): deterministic synthetic trees and records, and the
// dataset checksum.  Native C++, part of the product library so bench.py and
// users can build the canonical workloads without any test code.
//
//   st_synthetic_tree      generate_synthetic_tree   (synthetic.cpp:82-154)
//   st_synthetic_dataset   generate_synthetic_dataset (synthetic.cpp:156-182)
//   st_dataset_checksum    dataset_checksum           (dataset.cpp:76-93)
//   st_fnv1a64             FNV-1a-64 over raw bytes (label hashes)
//
// Same seed -> same tree / records as the reference on any standard library:
// draws come from std::mt19937_64 through the reference's bounded-draw rule.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/spectree_b200.h"

namespace st_internal {
void set_error(const std::string& msg);  // st_capi.cu: feeds st_last_error()
}

namespace {

constexpr uint32_t kGridBits = 23;  // threshold grid k / 2^23 (synthetic.cpp:17)
constexpr uint32_t kGrid = 1u << kGridBits;

inline uint64_t draw_below(std::mt19937_64& rng, uint64_t bound) {
  return static_cast<uint64_t>((static_cast<unsigned __int128>(rng()) * bound) >> 64);
}

struct Builder {
  // linked tree in flat arrays
  std::vector<uint32_t> attr;
  std::vector<float> thr;
  std::vector<int32_t> left, right;
  std::vector<int64_t> cls;

  int32_t add() {
    attr.push_back(0);
    thr.push_back(0.0f);
    left.push_back(-1);
    right.push_back(-1);
    cls.push_back(-1);
    return static_cast<int32_t>(attr.size() - 1);
  }
};

// A growing leaf: node id, depth, and its attribute box [lo, hi) on the grid
// (one row of `box` = lo[0..A) then hi[0..A)).
struct Frontier {
  uint32_t arity;
  std::vector<int32_t> node;
  std::vector<uint32_t> depth;
  std::vector<uint32_t> box;

  uint32_t* lo(size_t i) { return box.data() + i * 2 * arity; }
  uint32_t* hi(size_t i) { return lo(i) + arity; }
  bool wide(size_t i, uint32_t a) { return hi(i)[a] - lo(i)[a] >= 2; }
  bool splittable(size_t i) {
    for (uint32_t a = 0; a < arity; ++a)
      if (wide(i, a)) return true;
    return false;
  }
};

bool pick_wide(Frontier& f, size_t i, std::mt19937_64& rng, std::vector<uint32_t>& scratch,
               uint32_t* out) {
  scratch.clear();
  for (uint32_t a = 0; a < f.arity; ++a)
    if (f.wide(i, a)) scratch.push_back(a);
  if (scratch.empty()) return false;
  *out = scratch[draw_below(rng, scratch.size())];
  return true;
}

// Split frontier leaf i at its box midpoint on `a`: slot i becomes the left
// child, the right child is appended (synthetic.cpp:46-65).
void split(Builder& b, Frontier& f, size_t i, uint32_t a) {
  const uint32_t mid = f.lo(i)[a] + (f.hi(i)[a] - f.lo(i)[a]) / 2;
  const int32_t nd = f.node[i];
  const int32_t l = b.add();
  const int32_t r = b.add();
  b.cls[nd] = -1;
  b.attr[nd] = a;
  b.thr[nd] = static_cast<float>(mid) / static_cast<float>(kGrid);
  b.left[nd] = l;
  b.right[nd] = r;
  const size_t j = f.node.size();
  f.node.push_back(r);
  f.depth.push_back(f.depth[i] + 1);
  f.box.resize(f.box.size() + 2 * f.arity);
  std::memcpy(f.lo(j), f.lo(i), 2 * f.arity * sizeof(uint32_t));
  f.lo(j)[a] = mid;
  f.node[i] = l;
  f.depth[i] += 1;
  f.hi(i)[a] = mid;
}

}  // namespace

extern "C" {

int st_synthetic_tree(uint32_t depth, uint32_t leaves, uint32_t arity, uint32_t classes,
                      uint64_t seed, st_node* out, uint32_t cap, uint32_t* n_out) {
  auto err = [](const std::string& m) {
    st_internal::set_error(m);
    return (int)ST_ERR_ARGUMENT;
  };
  if (!n_out) return err("null n_out");
  if (arity == 0 || classes == 0) return err("arity and class count must be >= 1");
  if (depth == 0) {
    if (leaves != 1) return err("depth 0 admits exactly one leaf");
  } else {
    if (leaves < depth + 1)
      return err("leaf count " + std::to_string(leaves) + " cannot reach depth " +
                 std::to_string(depth) + "; need at least depth + 1 leaves");
    if (depth < 32 && (uint64_t)leaves > (1ull << depth))
      return err("leaf count " + std::to_string(leaves) + " exceeds 2^depth");
  }
  std::mt19937_64 rng(seed);
  Builder b;
  Frontier f{arity, {}, {}, {}};
  f.node.push_back(b.add());
  f.depth.push_back(0);
  f.box.assign(2 * arity, 0);
  for (uint32_t a = 0; a < arity; ++a) f.hi(0)[a] = kGrid;
  std::vector<uint32_t> scratch;
  const std::string exhausted = "requested shape exhausts the threshold grid; reduce depth";
  // spine: keep splitting slot 0 (the newest left child), rotating attributes
  for (uint32_t d = 0; d < depth; ++d) {
    uint32_t a = d % arity;
    if (!f.wide(0, a) && !pick_wide(f, 0, rng, scratch, &a)) return err(exhausted);
    split(b, f, 0, a);
  }
  // fill: uniformly drawn eligible leaf, uniformly drawn wide attribute
  std::vector<size_t> eligible;
  while (f.node.size() < leaves) {
    eligible.clear();
    for (size_t i = 0; i < f.node.size(); ++i)
      if (f.depth[i] < depth && f.splittable(i)) eligible.push_back(i);
    if (eligible.empty()) return err(exhausted);
    const size_t pick = eligible[draw_below(rng, eligible.size())];
    uint32_t a = 0;
    if (!pick_wide(f, pick, rng, scratch, &a)) return err(exhausted);
    split(b, f, pick, a);
  }
  for (size_t i = 0; i < f.node.size(); ++i) b.cls[f.node[i]] = (int64_t)draw_below(rng, classes);
  // breadth-first encoding (tree.cpp:72-113)
  const uint32_t n = (uint32_t)b.attr.size();
  *n_out = n;
  if (!out || cap < n) return ST_OK;
  std::vector<int32_t> q;
  q.reserve(n);
  q.push_back(0);
  uint32_t next_child = 1;
  for (size_t i = 0; i < q.size(); ++i) {
    const int32_t v = q[i];
    st_node e;
    if (b.left[v] < 0) {
      e = st_node{0u, INFINITY, (uint32_t)i, (uint32_t)b.cls[v]};
    } else {
      e = st_node{b.attr[v], b.thr[v], next_child, ST_NO_CLASS};
      q.push_back(b.left[v]);
      q.push_back(b.right[v]);
      next_child += 2;
    }
    out[i] = e;
  }
  return ST_OK;
}

int st_synthetic_dataset(uint64_t count, uint32_t arity, uint64_t seed, int gaussian, float* out) {
  if (arity == 0) {
    st_internal::set_error("dataset arity must be >= 1");
    return ST_ERR_ARGUMENT;
  }
  if (count && !out) {
    st_internal::set_error("null output");
    return ST_ERR_ARGUMENT;
  }
  std::mt19937_64 rng(seed);
  const uint64_t total = count * arity;
  if (!gaussian) {
    for (uint64_t i = 0; i < total; ++i) out[i] = static_cast<float>(rng() >> 40) * 0x1p-24f;
  } else {
    constexpr double kPi = 3.141592653589793238462643383279502884;
    for (uint64_t i = 0; i < total; ++i) {
      const double u1 = (static_cast<double>(rng() >> 40) + 1.0) * 0x1p-24;
      const double u2 = static_cast<double>(rng() >> 40) * 0x1p-24;
      const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
      out[i] = static_cast<float>(0.5 + 0.15 * z);
    }
  }
  return ST_OK;
}

uint64_t st_fnv1a64(const void* data, uint64_t n) {
  const auto* p = static_cast<const unsigned char*>(data);
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

uint64_t st_dataset_checksum(const float* x, uint64_t count, uint32_t arity) {
  uint64_t h = 0xcbf29ce484222325ull;
  auto mix = [&h](const void* d, uint64_t n) {
    const auto* p = static_cast<const unsigned char*>(d);
    for (uint64_t i = 0; i < n; ++i) {
      h ^= p[i];
      h *= 0x100000001b3ull;
    }
  };
  mix(&arity, sizeof arity);
  mix(&count, sizeof count);
  mix(x, count * arity * sizeof(float));
  return h;
}

}  // extern "C"

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
#include "st_internal.cuh"

namespace sti {
thread_local std::string g_error;
thread_local uint32_t g_launches = 0;
}  // namespace sti

namespace st_internal {
void set_error(const std::string& msg) { g_error = msg; }
void set_launches(uint32_t n) { g_launches = n; }
}  // namespace st_internal

namespace sti {
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

}  // namespace sti

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
    // Trees are folded (leaf pairs inside terminal nodes, fold_tree) when the
    // encoding allows: ~40 % fewer tree bytes to stream through the ring and
    // one node load fewer per walk that ends in a pair (C4).
    const bool fold = 4ull * maxattr < 1024 && !env_u32("ST_FOREST_NO_FOLD", 0);
    f->compact.reserve(total + t);
    std::vector<CNode> ft;
    for (uint32_t k = 0; k < t; ++k) {
      if (f->compact.size() & 1u) f->compact.push_back(CNode{0.0f, kLeafBit});  // 16-byte align
      f->offsets.push_back((uint32_t)f->compact.size());
      if (fold && sizes[k] > 1 && fold_tree(trees[k], sizes[k], f->abits, ft)) {
        f->compact.insert(f->compact.end(), ft.begin(), ft.end());
      } else {
        ft.clear();
        for (uint32_t i = 0; i < sizes[k]; ++i) {
          const st_node& nd = trees[k][i];
          if (nd.class_id != ST_NO_CLASS)
            ft.push_back(CNode{nd.threshold, kLeafBit | nd.class_id});
          else
            ft.push_back(CNode{nd.threshold, ((8u * nd.child) << f->abits) | (4u * nd.attribute)});
        }
        f->compact.insert(f->compact.end(), ft.begin(), ft.end());
      }
      const uint32_t tb = (uint32_t)((ft.size() * sizeof(CNode) + 15) & ~size_t(15));
      f->tree_bytes.push_back(tb);
      f->max_tree_bytes = std::max(f->max_tree_bytes, tb);
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

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
//   * the host-buffer path (chunked H2D / kernel / D2H over three streams) and
//     the sample-sharded multi-GPU driver.
#include <pthread.h>

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

// depths != null: the data kernel also writes traversal depths (the algorithm
// field is then ignored).
void eval_device_impl(st_tree* t, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
                      const st_geom* geom, uint32_t* labels, st_stats* stats, cudaStream_t s,
                      uint32_t* depths = nullptr) {
  if (!t) fail(ST_ERR_ARGUMENT, "null tree");
  check_common(m, a, ld, layout, t->info.max_attribute);
  st_geom g{};
  if (geom) g = *geom;
  const uint32_t algo = depths ? (uint32_t)ST_ALGO_DATA : resolve_algo(t, g, stats != nullptr);
  if (stats && algo != ST_ALGO_SPECULATIVE)
    fail(ST_ERR_ARGUMENT, "per-record stats are produced by the speculative kernel only");
  if (m == 0) return;  // empty dataset: empty output, no launch
  if (!x || !labels) fail(ST_ERR_ARGUMENT, "null data or label pointer");
  const int dev = current_device();
  if (algo == ST_ALGO_DATA)
    eval_data_device(t, x, m, a, ld, layout, g, labels, depths, s, dev);
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

// Host worker threads for packing pageable records into pinned staging: the
// driver's own pageable H2D stages through one thread (~11 GB/s on the B200
// boxes); several threads copying into pinned buffers keep PCIe busy.  Jobs
// from concurrent callers share the workers; the caller runs part 0 itself.
class HostCopyPool {
 public:
  static HostCopyPool& get() {
    static HostCopyPool* p = [] {
      auto* q = new HostCopyPool();  // intentionally leaked (detached workers)
      // a fork()ed child has no workers: run its jobs on the caller alone
      pthread_atfork(nullptr, nullptr, [] { reset_after_fork(); });
      return q;
    }();
    instance() = p;
    return *p;
  }
  int width() const { return (int)workers_ + 1; }
  // fn(i) for i in [0, n); returns when all parts are done.  Parts are
  // claimed from a shared counter by the caller and up to n - 1 woken
  // workers, so a descheduled worker delays at most the part it holds.
  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 1 || workers_ == 0) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    struct Job {
      std::atomic<int> next{0}, done{0};
      int n = 0;
      std::mutex mu;
      std::condition_variable cv;
    };
    auto job = std::make_shared<Job>();
    job->n = n;
    const std::function<void(int)>* f = &fn;  // valid while any part is unclaimed
    auto work = [job, f] {
      for (int i; (i = job->next.fetch_add(1)) < job->n;) {
        (*f)(i);
        if (job->done.fetch_add(1) + 1 == job->n) {
          std::lock_guard<std::mutex> lk(job->mu);
          job->cv.notify_all();
        }
      }
    };
    const int helpers = std::min<int>((int)workers_, n - 1);
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (int h = 0; h < helpers; ++h) q_.emplace_back(work);
    }
    if (helpers == 1) cv_.notify_one();
    else cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(job->mu);
    job->cv.wait(lk, [&] { return job->done.load() == job->n; });
  }

 private:
  static HostCopyPool*& instance() {
    static HostCopyPool* i = nullptr;
    return i;
  }
  static void reset_after_fork() {
    HostCopyPool* p = instance();
    if (!p) return;
    p->workers_ = 0;
    new (&p->mu_) std::mutex();  // may have been held by a thread that is gone
    new (&p->cv_) std::condition_variable();
    new (&p->q_) std::deque<std::function<void()>>();  // drop (leak) the parent's queue
  }
  HostCopyPool() {
    const uint32_t hw = std::max(1u, std::thread::hardware_concurrency());
    // read once, when the pool is first used (process-wide width of the
    // host packing threads; never consulted on the launch path)
    const char* env = std::getenv("ST_HOST_COPY_THREADS");
    workers_ = (env && *env ? (uint32_t)std::strtoul(env, nullptr, 10) : std::min(16u, hw)) - 1u;
    if (workers_ > 63) workers_ = 0;  // ST_HOST_COPY_THREADS=0 -> single-threaded
    for (uint32_t i = 0; i < workers_; ++i)
      std::thread([this] {
        for (;;) {
          std::function<void()> task;
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return !q_.empty(); });
            task = std::move(q_.front());
            q_.pop_front();
          }
          task();
        }
      }).detach();
  }
  uint32_t workers_ = 0;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
};

// Pack records [r0, r0 + rows) of host x into dst as the dense device layout
// the kernels get from the host path (AoS: rows x a; SoA: a columns of rows),
// split over the copy pool (byte ranges of a contiguous block, else row ranges).
void pack_records(void* dst, const float* x, uint64_t r0, uint64_t rows, uint32_t a, uint64_t ld,
                  int layout) {
  HostCopyPool& pool = HostCopyPool::get();
  const uint64_t row_bytes = (uint64_t)a * 4;
  const uint64_t bytes = rows * row_bytes;
  // ~512 KB parts, claimed dynamically by the pool's threads
  const int parts = (int)std::max<uint64_t>(1, std::min<uint64_t>(4096, bytes >> 19));
  char* d = static_cast<char*>(dst);
  if (layout == ST_LAYOUT_AOS && ld == a) {
    const char* src = reinterpret_cast<const char*>(x + r0 * a);
    const uint64_t piece = ((bytes + parts - 1) / parts + 4095) & ~uint64_t(4095);
    pool.run(parts, [&](int i) {
      const uint64_t b0 = std::min(bytes, (uint64_t)i * piece), b1 = std::min(bytes, b0 + piece);
      if (b1 > b0) std::memcpy(d + b0, src + b0, b1 - b0);
    });
    return;
  }
  const uint64_t per = (rows + parts - 1) / parts;
  pool.run(parts, [&](int i) {
    const uint64_t q0 = std::min(rows, (uint64_t)i * per), q1 = std::min(rows, q0 + per);
    if (layout == ST_LAYOUT_AOS) {
      for (uint64_t r = q0; r < q1; ++r) std::memcpy(d + r * row_bytes, x + (r0 + r) * ld, row_bytes);
    } else {
      for (uint32_t k = 0; k < a; ++k)
        std::memcpy(d + ((uint64_t)k * rows + q0) * 4, x + (uint64_t)k * ld + r0 + q0, (q1 - q0) * 4);
    }
  });
}

// Per-device staging slots reused across host-path calls (a slot = stream +
// device record/label buffers + pinned label staging + pinned record staging
// for pageable inputs), so the H2D/kernel/D2H pipeline does not pay
// cudaMalloc/cudaFree or page pinning per call.
struct Slot {
  cudaStream_t stream = nullptr;
  float* x = nullptr;
  size_t x_cap = 0;
  uint32_t* out[3] = {nullptr, nullptr, nullptr};  // labels + up to 2 counters
  uint32_t* pinned[3] = {nullptr, nullptr, nullptr};
  size_t out_cap = 0;
  void* pin_x = nullptr;  // pinned record staging (pageable inputs)
  size_t pin_cap = 0;
  cudaEvent_t x_free = nullptr;  // recorded after the last copy out of pin_x / into pinned[0]
  bool busy = false;
};

class SlotPool {
 public:
  std::vector<Slot*> acquire(int dev, int n, size_t x_bytes, size_t rows, size_t pin_bytes = 0) {
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
        if (sl->pin_cap < pin_bytes) {
          cudaFreeHost(sl->pin_x);
          sl->pin_x = nullptr;
          sl->pin_cap = 0;
          CK(cudaMallocHost(&sl->pin_x, pin_bytes));
          sl->pin_cap = pin_bytes;
        }
        if (!sl->x_free) CK(cudaEventCreateWithFlags(&sl->x_free, cudaEventDisableTiming));
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

// Stream-ordered device memory for st_eval_timed's per-call buffers: one pool
// per device that keeps freed memory (release threshold = max), so a call's
// allocation after the first is a pool hit rather than cudaMalloc/cudaFree.
cudaMemPool_t timed_pool(int dev) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lk(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool;
  CK(cudaMemPoolCreate(&pool, &props));
  uint64_t keep = UINT64_MAX;
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  pools[dev] = pool;
  return pool;
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
  // pageable records go through pinned staging packed by the host copy pool
  const bool staged = !is_pinned_or_device(x);
  std::vector<Slot*> slots =
      slot_pool().acquire(dev, ns, chunk * row_bytes, chunk, staged ? chunk * row_bytes : 0);
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
      pack_records(outs[k] + pending[i].first, reinterpret_cast<const float*>(slots[i]->pinned[k]), 0,
                   pending[i].second, 1, 1, ST_LAYOUT_AOS);
    pending[i] = {0, 0};
  };
  for (uint64_t c = 0; c < n_chunks; ++c) {
    const int i = (int)(c % ns);
    Slot* sl = slots[i];
    drain(i);
    const uint64_t r0 = c * chunk;
    const uint64_t rows = std::min(chunk, m - r0);
    if (staged) {
      // the previous H2D out of this slot's pinned buffer must be done; the
      // other slots' copies and kernels run while this chunk is packed
      CK(cudaEventSynchronize(sl->x_free));
      pack_records(sl->pin_x, x, r0, rows, a, ld, layout);
      CK(cudaMemcpyAsync(sl->x, sl->pin_x, rows * row_bytes, cudaMemcpyHostToDevice, sl->stream));
      CK(cudaEventRecord(sl->x_free, sl->stream));
    } else if (layout == ST_LAYOUT_AOS) {
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
    // Layout 0 folds trees (leaf pairs inside terminal nodes, fold_tree) when
    // the encoding allows: ~40 % fewer tree bytes to stream through the ring
    // and one node load fewer per walk that ends in a pair (C4).  Layout 1
    // keeps every tree plain (ST_VAR_NO_FOLD).
    for (int l = 0; l < 2; ++l) {
      st_forest::Layout& L = f->lay[l];
      const bool fold = l == 0 && 4ull * maxattr < 1024;
      L.compact.reserve(total + t);
      std::vector<CNode> ft;
      for (uint32_t k = 0; k < t; ++k) {
        if (L.compact.size() & 1u) L.compact.push_back(CNode{0.0f, kLeafBit});  // 16-byte align
        L.offsets.push_back((uint32_t)L.compact.size());
        if (fold && sizes[k] > 1 && fold_tree(trees[k], sizes[k], f->abits, ft)) {
          L.compact.insert(L.compact.end(), ft.begin(), ft.end());
        } else {
          ft.clear();
          for (uint32_t i = 0; i < sizes[k]; ++i) {
            const st_node& nd = trees[k][i];
            if (nd.class_id != ST_NO_CLASS)
              ft.push_back(CNode{nd.threshold, kLeafBit | nd.class_id});
            else
              ft.push_back(CNode{nd.threshold, ((8u * nd.child) << f->abits) | (4u * nd.attribute)});
          }
          L.compact.insert(L.compact.end(), ft.begin(), ft.end());
        }
        const uint32_t tb = (uint32_t)((ft.size() * sizeof(CNode) + 15) & ~size_t(15));
        L.tree_bytes.push_back(tb);
        L.max_tree_bytes = std::max(L.max_tree_bytes, tb);
      }
      if (L.compact.size() & 1u) L.compact.push_back(CNode{0.0f, kLeafBit});
      L.compact.push_back(CNode{0.0f, kLeafBit});  // tail padding for the last 16-byte copy
      L.offsets.push_back((uint32_t)L.compact.size());
    }
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

}  // extern "C"

namespace sti {
// st_eval / st_eval_depths: the host-buffer pipeline around eval_device_impl
// (stats and depths come back beside the labels, through the same slots).
void eval_host(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
               const st_geom* geom, uint32_t* labels, st_stats* stats, uint32_t* depths) {
  g_launches = 0;
  st_tree* t = const_cast<st_tree*>(tree);
  if (!t) fail(ST_ERR_ARGUMENT, "null tree");
  uint64_t ld2 = ld;
  check_common(m, a, ld2, layout, t->info.max_attribute);
  st_geom g{};
  if (geom) g = *geom;
  if (!depths) resolve_algo(t, g, stats != nullptr);
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
  if (depths) extra.push_back({depths, nullptr});
  uint32_t launches = 0;
  host_pipeline(x, m, a, ld2, layout, labels, extra,
                [&](const float* xd, uint64_t rows, uint64_t ldd, uint32_t* lab,
                    std::vector<uint32_t*>& ex, cudaStream_t s) {
                  st_stats sd{};
                  if (stats) {
                    sd.iterations = ex[0];
                    sd.doubling_steps = ex[1];
                  }
                  eval_device_impl(t, xd, rows, a, ldd, layout, &g, lab, stats ? &sd : nullptr, s,
                                   depths ? ex.back() : nullptr);
                  launches += g_launches;
                  g_launches = 0;
                });
  g_launches = launches;
}
}  // namespace sti

extern "C" {

int st_eval(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld, int layout,
            const st_geom* geom, uint32_t* labels, st_stats* stats) {
  return guarded([&] { eval_host(tree, x, m, a, ld, layout, geom, labels, stats, nullptr); });
}

int st_eval_depths(const st_tree* tree, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                   int layout, const st_geom* geom, uint32_t* labels, uint32_t* depths) {
  return guarded([&] {
    if (m && !depths) fail(ST_ERR_ARGUMENT, "null depth output");
    eval_host(tree, x, m, a, ld, layout, geom, labels, nullptr, depths);
  });
}

int st_eval_depths_device(const st_tree* tree, const float* x, uint64_t m, uint32_t a,
                          uint64_t ld, int layout, const st_geom* geom, uint32_t* labels,
                          uint32_t* depths, void* stream) {
  return guarded([&] {
    g_launches = 0;
    if (m && !depths) fail(ST_ERR_ARGUMENT, "null depth output");
    eval_device_impl(const_cast<st_tree*>(tree), x, m, a, ld, layout, geom, labels, nullptr,
                     static_cast<cudaStream_t>(stream), depths);
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
    const int dev = current_device();
    const uint64_t row_bytes = (uint64_t)a * 4;
    // pageable records: chunks (total / 8, 2..64 MB) packed into two pinned
    // staging buffers by the host copy pool while the previous chunk is on
    // the wire
    const bool staged = !is_pinned_or_device(x);
    const uint64_t cbytes = std::min<uint64_t>(64ull << 20, std::max<uint64_t>(2ull << 20, m * row_bytes / 8));
    const uint64_t chunk = std::min<uint64_t>(m, std::max<uint64_t>(256, cbytes / row_bytes));
    const bool staged_out = !is_pinned_or_device(labels);
    std::vector<Slot*> stage;
    if (staged || staged_out)
      stage = slot_pool().acquire(dev, 2, 0, staged_out ? chunk : 0, staged ? chunk * row_bytes : 0);
    struct Release {
      std::vector<Slot*>& s;
      ~Release() {
        for (Slot* sl : s) cudaEventSynchronize(sl->x_free);
        if (!s.empty()) slot_pool().release(s);
      }
    } release{stage};
    cudaMemPool_t pool = timed_pool(dev);
    const auto o0 = Clock::now();
    float* xd = nullptr;
    uint32_t* ld_out = nullptr;
    CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&xd), m * row_bytes, pool, ev.s));
    struct Free {
      void* p[2];
      cudaStream_t s;
      ~Free() {
        for (void* q : p)
          if (q) cudaFreeAsync(q, s);
        cudaStreamSynchronize(s);
      }
    } guard{{xd, nullptr}, ev.s};
    CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&ld_out), m * 4, pool, ev.s));
    guard.p[1] = ld_out;
    const auto a1 = Clock::now();
    CK(cudaEventRecord(ev.e[0], ev.s));
    if (staged) {
      for (uint64_t r0 = 0, c = 0; r0 < m; r0 += chunk, ++c) {
        Slot* sl = stage[c & 1];
        const uint64_t rows = std::min(chunk, m - r0);
        CK(cudaEventSynchronize(sl->x_free));
        pack_records(sl->pin_x, x, r0, rows, a, ld2, layout);
        if (layout == ST_LAYOUT_AOS)
          CK(cudaMemcpyAsync(xd + r0 * a, sl->pin_x, rows * row_bytes, cudaMemcpyHostToDevice, ev.s));
        else
          CK(cudaMemcpy2DAsync(xd + r0, m * 4, sl->pin_x, rows * 4, rows * 4, a, cudaMemcpyHostToDevice,
                               ev.s));
        CK(cudaEventRecord(sl->x_free, ev.s));
      }
    } else if (layout == ST_LAYOUT_AOS) {
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
    if (staged_out) {
      // pageable labels: chunks land in the two pinned label buffers; chunk
      // c - 1 is copied out by the host pool while chunk c is on the wire
      uint64_t prev0 = 0, prev_rows = 0;
      int prev_k = 0;
      auto copy_out = [&](int k, uint64_t r0, uint64_t rows) {
        CK(cudaEventSynchronize(stage[k]->x_free));
        pack_records(labels + r0, reinterpret_cast<const float*>(stage[k]->pinned[0]), 0, rows, 1, 1,
                     ST_LAYOUT_AOS);
      };
      for (uint64_t r0 = 0, c = 0; r0 < m; r0 += chunk, ++c) {
        const int k = (int)(c & 1);
        const uint64_t rows = std::min(chunk, m - r0);
        CK(cudaMemcpyAsync(stage[k]->pinned[0], ld_out + r0, rows * 4, cudaMemcpyDeviceToHost, ev.s));
        CK(cudaEventRecord(stage[k]->x_free, ev.s));
        if (prev_rows) copy_out(prev_k, prev0, prev_rows);
        prev0 = r0, prev_rows = rows, prev_k = k;
      }
      CK(cudaEventRecord(ev.e[3], ev.s));
      copy_out(prev_k, prev0, prev_rows);
    } else {
      CK(cudaMemcpyAsync(labels, ld_out, m * 4, cudaMemcpyDefault, ev.s));
      CK(cudaEventRecord(ev.e[3], ev.s));
    }
    CK(cudaStreamSynchronize(ev.s));
    const auto f0 = Clock::now();
    guard.p[0] = guard.p[1] = nullptr;
    CK(cudaFreeAsync(xd, ev.s));
    CK(cudaFreeAsync(ld_out, ev.s));
    CK(cudaStreamSynchronize(ev.s));
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
                          uint64_t ld, int layout, const st_geom* geom, uint32_t* labels,
                          void* stream) {
  return guarded([&] {
    g_launches = 0;
    st_geom g{};
    if (geom) g = *geom;
    forest_device_impl(const_cast<st_forest*>(forest), x, m, a, ld, layout, g, labels,
                       static_cast<cudaStream_t>(stream));
  });
}

int st_forest_eval(const st_forest* forest, const float* x, uint64_t m, uint32_t a, uint64_t ld,
                   int layout, const st_geom* geom, uint32_t* labels) {
  return guarded([&] {
    g_launches = 0;
    st_forest* f = const_cast<st_forest*>(forest);
    if (!f) fail(ST_ERR_ARGUMENT, "null forest");
    uint64_t ld2 = ld;
    check_common(m, a, ld2, layout, f->max_attribute);
    if (m == 0) return;
    if (!x || !labels) fail(ST_ERR_ARGUMENT, "null data or label pointer");
    current_device();
    st_geom g{};
    if (geom) g = *geom;
    uint32_t launches = 0;
    host_pipeline(x, m, a, ld2, layout, labels, {},
                  [&](const float* xd, uint64_t rows, uint64_t ldd, uint32_t* lab,
                      std::vector<uint32_t*>&, cudaStream_t s) {
                    forest_device_impl(f, xd, rows, a, ldd, layout, g, lab, s);
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

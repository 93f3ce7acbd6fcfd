// Resident frame-stream evaluator (st_frames_*, include/spectree_b200.h).
//
// A video-rate caller (C3: one 1920x1080 frame of 8 features per pixel)
// classifies one frame after another.  One launch per frame pays a launch,
// the tree staging and the record pipeline's ramp-up every time (C3: ~25 us
// per single-frame launch against ~18 us per frame inside a 32-frame launch).
// Here one k_data<FRAMES> grid stays resident: the tree is staged once, and
// the frames published into a device ring of `ring` slots form one
// continuous tile sequence that every warp walks with its usual stride, the
// stage refill running across frame boundaries; per frame the only
// synchronisation is a counter the producer's stream writes
// (cuStreamWriteValue32) and a per-slot count of walked tiles the kernel
// adds to (release reductions) for consumers to wait on
// (cuStreamWaitValue64 or host polling).  No grid barrier anywhere.  The reference has no frame API; the
// per-frame result is exactly eval_serial's labels (eval_serial.cpp:33-41).
#include <chrono>
#include <thread>

#include "st_internal.cuh"

namespace sti {

using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValue64Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

template <class F>
static F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    fail(ST_ERR_CUDA, std::string("driver entry point ") + name + " unavailable (stream memory operations)");
  }
  return reinterpret_cast<F>(p);
}

static WriteValue32Fn write_value32() {
  static WriteValue32Fn f = driver_fn<WriteValue32Fn>("cuStreamWriteValue32");
  return f;
}
static WaitValue64Fn wait_value64() {
  static WaitValue64Fn f = driver_fn<WaitValue64Fn>("cuStreamWaitValue64");
  return f;
}

static void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) fail(ST_ERR_CUDA, std::string(what) + " failed (CUresult " + std::to_string(r) + ")");
}

// ---- launch: k_data<..., FRAMES = true> for the planned walk -----------------
// returns the grid's warp count (a frame is done when that many warps counted it)
template <int A, int S, int TLOC>
static uint64_t launch_frames_t(const DataArgs& d, const Staging& stg, size_t smem, int dev, uint32_t bps,
                                uint32_t max_ctas, cudaStream_t s) {
  auto fn = k_data<A, S, TLOC, kTma, 1, false, true>;
  const uint64_t n_tiles = (d.p.m + 32 * S - 1) / (32 * S);
  int blocks = blocks_for((const void*)fn, smem, dev, bps, n_tiles, stg.warps);
  if (max_ctas) blocks = std::min<int>(blocks, (int)max_ctas);
  static const ConstTree<1> dummy{};
  clear_stale_error();
  fn<<<blocks, stg.warps * 32, smem, s>>>(d, stg.tmap, dummy);
  check_launch();
  return (uint64_t)blocks * stg.warps;
}

template <int A, int S>
static uint64_t launch_frames_tloc(int tloc, const DataArgs& d, const Staging& stg, size_t smem, int dev,
                               uint32_t bps, uint32_t max_ctas, cudaStream_t s) {
  if (tloc == ST_TREE_SHARED) {
    if constexpr (A == 8 || A == 16) {
      if (d.record_regs == 2) return launch_frames_t<A, S, kSharedT>(d, stg, smem, dev, bps, max_ctas, s);
      if (d.record_regs) return launch_frames_t<A, S, kSharedReg>(d, stg, smem, dev, bps, max_ctas, s);
    }
    return launch_frames_t<A, S, kShared>(d, stg, smem, dev, bps, max_ctas, s);
  }
  return launch_frames_t<A, S, kGlobal>(d, stg, smem, dev, bps, max_ctas, s);
}

template <int A>
static uint64_t launch_frames_a(int tloc, const DataArgs& d, const Staging& stg, size_t smem, int dev,
                            uint32_t bps, uint32_t max_ctas, cudaStream_t s) {
  if constexpr (A == 8 || A == 16) {
    if (stg.S == 4) return launch_frames_tloc<A, 4>(tloc, d, stg, smem, dev, bps, max_ctas, s);
  }
  if (stg.S == 2) return launch_frames_tloc<A, 2>(tloc, d, stg, smem, dev, bps, max_ctas, s);
  return launch_frames_tloc<A, 1>(tloc, d, stg, smem, dev, bps, max_ctas, s);
}

}  // namespace sti

using namespace sti;

struct st_frames {
  st_tree* tree = nullptr;
  int dev = 0;
  uint64_t rpf = 0;  // records per frame
  uint32_t a = 0, ring = 0;
  float* x = nullptr;         // ring x rpf x a
  uint32_t* labels = nullptr; // ring x rpf
  uint32_t* ctl = nullptr;    // {published, closed_at, error, pad}, uint64 done[ring] (k_data<FRAMES>)
  uint64_t tiles = 0;         // record tiles per frame: frame seq done at done[slot] >= (seq / ring + 1) * tiles
  uint64_t* host_word = nullptr;  // pinned: polled control words
  cudaStream_t ks = nullptr, cs = nullptr;  // resident kernel, host-convenience copies
  uint32_t next_pub = 0;
  uint64_t timeout_ms = 0;
  std::mutex mu;

  CUdeviceptr word(uint32_t i) const { return reinterpret_cast<CUdeviceptr>(ctl + i); }
  CUdeviceptr done_word(uint64_t seq) const { return word(kFDone + 2 * slot(seq)); }
  uint64_t done_target(uint64_t seq) const { return (seq / ring + 1) * tiles; }
  uint32_t slot(uint64_t seq) const { return (uint32_t)(seq % ring); }
  // one control word read through the copy stream (no device-wide sync)
  uint64_t read_word(uint32_t i, size_t bytes = 4) {
    *host_word = 0;
    CK(cudaMemcpyAsync(host_word, ctl + i, bytes, cudaMemcpyDeviceToHost, cs));
    CK(cudaStreamSynchronize(cs));
    return *host_word;
  }
  // host-side wait until frame seq is done, bounded by the idle timeout
  void host_wait_done(uint64_t seq, const char* what) {
    const auto t0 = std::chrono::steady_clock::now();
    while (true) {
      if (read_word(kFDone + 2 * slot(seq), 8) >= done_target(seq)) return;
      if (read_word(kFError)) fail(ST_ERR_CUDA, std::string(what) + ": frame stream stopped (idle timeout)");
      if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms))
        fail(ST_ERR_CUDA, std::string(what) + ": timed out waiting for frame " + std::to_string(seq));
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }
};

extern "C" {

int st_frames_open(const st_tree* tree, uint64_t records, uint32_t a, uint32_t ring, const st_geom* geom,
                   uint32_t max_ctas, uint32_t idle_timeout_ms, st_frames** out) {
  return guarded([&] {
    if (!out) fail(ST_ERR_ARGUMENT, "null output handle");
    *out = nullptr;
    if (!tree) fail(ST_ERR_ARGUMENT, "null tree");
    if (a != 8 && a != 16 && a != 32)
      fail(ST_ERR_ARGUMENT, "frame streams take 8, 16 or 32 attributes per record (TMA row-local tiles)");
    if (records == 0) fail(ST_ERR_ARGUMENT, "records per frame must be >= 1");
    if (ring == 0 || ring > 4096) fail(ST_ERR_ARGUMENT, "ring must hold 1..4096 frames");
    uint64_t ld = a;
    check_common(records, a, ld, ST_LAYOUT_AOS, tree->info.max_attribute);
    if ((uint64_t)ring * records * a / 32 >= (1ull << 31))
      fail(ST_ERR_ARGUMENT, "frame ring too large for one tensor map");
    st_geom g{};
    if (geom) g = *geom;
    if (g.algo != ST_ALGO_AUTO && g.algo != ST_ALGO_DATA && g.algo != ST_ALGO_SPECULATIVE)
      fail(ST_ERR_ARGUMENT, "unknown algorithm " + std::to_string(g.algo));
    if (g.tree_loc == ST_TREE_CONSTANT) g.tree_loc = ST_TREE_AUTO;
    const int dev = current_device();
    std::unique_ptr<st_frames> f(new st_frames());
    f->tree = const_cast<st_tree*>(tree);
    f->dev = dev;
    f->rpf = records;
    f->a = a;
    f->ring = ring;
    f->timeout_ms = idle_timeout_ms ? idle_timeout_ms : 10000u;
    auto cleanup = [&] {
      cudaFree(f->x);
      cudaFree(f->labels);
      cudaFree(f->ctl);
      cudaFreeHost(f->host_word);
      if (f->ks) cudaStreamDestroy(f->ks);
      if (f->cs) cudaStreamDestroy(f->cs);
    };
    try {
      CK(cudaMalloc(reinterpret_cast<void**>(&f->x), (size_t)ring * records * a * 4));
      CK(cudaMalloc(reinterpret_cast<void**>(&f->labels), (size_t)ring * records * 4));
      CK(cudaMalloc(reinterpret_cast<void**>(&f->ctl), (4 + 2 * (size_t)ring) * 4));  // 16-byte aligned
      CK(cudaMallocHost(reinterpret_cast<void**>(&f->host_word), 64));
      CK(cudaStreamCreateWithFlags(&f->ks, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&f->cs, cudaStreamNonBlocking));
      std::vector<uint32_t> init(4 + 2 * (size_t)ring, 0u);
      init[kFClosed] = 0xFFFFFFFFu;
      CK(cudaMemcpy(f->ctl, init.data(), init.size() * 4, cudaMemcpyHostToDevice));
      (void)write_value32();
      (void)wait_value64();

      if (g.algo == ST_ALGO_SPECULATIVE) {
        // the speculative ring in frame mode (st_spec.cu: k_spec_ring<..., FR>)
        SpecFrames sf;
        sf.fctl = f->ctl;
        sf.ring = ring;
        sf.max_ctas = max_ctas;
        sf.ring_records = (uint64_t)ring * records;
        sf.idle_ns = (uint64_t)f->timeout_ms * 1000000ull;
        eval_spec_device(f->tree, f->x, records, a, a, ST_LAYOUT_AOS, g, f->labels, nullptr, f->ks, dev, &sf);
        f->tiles = sf.tiles;
        *out = f.release();
        return;
      }
      // the one-frame data plan (not a small input: the walk geometry of a
      // stream of frames), then a tensor map over the whole ring
      DataPlan pl = plan_data(f->tree, f->x, records, a, a, ST_LAYOUT_AOS, g, f->labels, nullptr, dev);
      if (pl.stg.loader != kTma) fail(ST_ERR_ARGUMENT, "frame stream needs TMA-staged records");
      if (pl.tloc != ST_TREE_SHARED && pl.tloc != ST_TREE_GLOBAL)
        fail(ST_ERR_ARGUMENT, "frame stream needs the compact node format (tree indices too large)");
      const uint64_t R = 32ull * pl.stg.S;
      if (records % R != 0)
        fail(ST_ERR_ARGUMENT, "records per frame must be a multiple of " + std::to_string(R) +
                                  " (whole record tiles per frame)");
      make_tmap(pl.stg, f->x, (uint64_t)ring * records, a);
      f->tiles = records / R;
      DataArgs d = pl.d;
      d.pdl = 0;
      d.fctl = f->ctl;
      d.ring = ring;
      d.frame_rows = (uint32_t)(records * a / 32);
      d.idle_ns = (uint64_t)f->timeout_ms * 1000000ull;
      switch (a) {
        case 8: launch_frames_a<8>(pl.tloc, d, pl.stg, pl.smem, dev, pl.bps, max_ctas, f->ks); break;
        case 16: launch_frames_a<16>(pl.tloc, d, pl.stg, pl.smem, dev, pl.bps, max_ctas, f->ks); break;
        default: launch_frames_a<32>(pl.tloc, d, pl.stg, pl.smem, dev, pl.bps, max_ctas, f->ks); break;
      }
    } catch (...) {
      cleanup();
      throw;
    }
    *out = f.release();
  });
}

int st_frames_slot(st_frames* f, uint64_t seq, float** records, uint32_t** labels) {
  return guarded([&] {
    if (!f) fail(ST_ERR_ARGUMENT, "null frame stream");
    const uint32_t s = f->slot(seq);
    if (records) *records = f->x + (size_t)s * f->rpf * f->a;
    if (labels) *labels = f->labels + (size_t)s * f->rpf;
  });
}

int st_frames_acquire(st_frames* f, uint64_t seq, void* stream) {
  return guarded([&] {
    if (!f) fail(ST_ERR_ARGUMENT, "null frame stream");
    if (seq < f->ring) return;  // the slot has never held a frame
    cu_check(wait_value64()(reinterpret_cast<CUstream>(stream), f->done_word(seq), f->done_target(seq - f->ring),
                            CU_STREAM_WAIT_VALUE_GEQ),
             "cuStreamWaitValue64");
  });
}

int st_frames_publish(st_frames* f, uint64_t seq, void* stream) {
  return guarded([&] {
    if (!f) fail(ST_ERR_ARGUMENT, "null frame stream");
    std::lock_guard<std::mutex> lk(f->mu);
    // publishing frame seq publishes every earlier frame too (one write per batch)
    if (seq < f->next_pub)
      fail(ST_ERR_ARGUMENT, "frames are published in order: frame " + std::to_string(seq) +
                                " is already published (next is " + std::to_string(f->next_pub) + ")");
    if (seq + 1 >= 0xFFFFFFFFull) fail(ST_ERR_ARGUMENT, "frame sequence exhausted (2^32 - 2 frames)");
    cu_check(write_value32()(reinterpret_cast<CUstream>(stream), f->word(kFPublished), (cuuint32_t)(seq + 1),
                             CU_STREAM_WRITE_VALUE_DEFAULT),
             "cuStreamWriteValue32");
    f->next_pub = (uint32_t)(seq + 1);
  });
}

int st_frames_wait(st_frames* f, uint64_t seq, void* stream) {
  return guarded([&] {
    if (!f) fail(ST_ERR_ARGUMENT, "null frame stream");
    cu_check(wait_value64()(reinterpret_cast<CUstream>(stream), f->done_word(seq), f->done_target(seq),
                            CU_STREAM_WAIT_VALUE_GEQ),
             "cuStreamWaitValue64");
  });
}

int st_frames_push(st_frames* f, const float* host_records, uint64_t* seq_out) {
  return guarded([&] {
    if (!f || !host_records) fail(ST_ERR_ARGUMENT, "null frame stream or records");
    std::lock_guard<std::mutex> lk(f->mu);
    const uint64_t seq = f->next_pub;
    if (seq >= f->ring) f->host_wait_done(seq - f->ring, "st_frames_push");
    const uint32_t s = f->slot(seq);
    CK(cudaMemcpyAsync(f->x + (size_t)s * f->rpf * f->a, host_records, (size_t)f->rpf * f->a * 4,
                       cudaMemcpyHostToDevice, f->cs));
    cu_check(write_value32()(f->cs, f->word(kFPublished), (cuuint32_t)(seq + 1), CU_STREAM_WRITE_VALUE_DEFAULT),
             "cuStreamWriteValue32");
    ++f->next_pub;
    if (seq_out) *seq_out = seq;
  });
}

int st_frames_pop(st_frames* f, uint64_t seq, uint32_t* host_labels) {
  return guarded([&] {
    if (!f || !host_labels) fail(ST_ERR_ARGUMENT, "null frame stream or labels");
    std::lock_guard<std::mutex> lk(f->mu);
    if (seq >= f->next_pub) fail(ST_ERR_ARGUMENT, "frame " + std::to_string(seq) + " was not published");
    if (seq + f->ring < f->next_pub)
      fail(ST_ERR_ARGUMENT, "frame " + std::to_string(seq) + " was overwritten by frame " +
                                std::to_string(seq + f->ring) + " (pop before publishing ring frames more)");
    f->host_wait_done(seq, "st_frames_pop");
    CK(cudaMemcpyAsync(host_labels, f->labels + (size_t)f->slot(seq) * f->rpf, (size_t)f->rpf * 4,
                       cudaMemcpyDeviceToHost, f->cs));
    CK(cudaStreamSynchronize(f->cs));
  });
}

int st_frames_status(st_frames* f, uint64_t* published, uint32_t* stopped) {
  return guarded([&] {
    if (!f) fail(ST_ERR_ARGUMENT, "null frame stream");
    if (published) *published = f->next_pub;
    if (stopped) *stopped = f->read_word(kFError);
  });
}

int st_frames_close(st_frames* f) {
  return guarded([&] {
    if (!f) return;
    std::unique_ptr<st_frames> own(f);
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(f->dev);
    // frames published so far are walked, then every warp meets closed_at
    const CUresult r = write_value32()(f->cs, f->word(kFClosed), (cuuint32_t)f->next_pub,
                                       CU_STREAM_WRITE_VALUE_DEFAULT);
    cudaError_t e1 = cudaStreamSynchronize(f->cs);
    cudaError_t e2 = cudaStreamSynchronize(f->ks);
    cudaFree(f->x);
    cudaFree(f->labels);
    cudaFree(f->ctl);
    cudaFreeHost(f->host_word);
    cudaStreamDestroy(f->ks);
    cudaStreamDestroy(f->cs);
    if (cur >= 0) cudaSetDevice(cur);
    cu_check(r, "cuStreamWriteValue32");
    CK(e1);
    CK(e2);
  });
}

}  // extern "C"

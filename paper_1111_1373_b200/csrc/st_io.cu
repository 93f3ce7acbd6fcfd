// Record / label files at scale and the streaming file -> GPU evaluator
// (SURVEY §8f row 3).  Formats are specified in include/spectree_b200.h.
//
// The reference reads datasets only as CSV (io.cpp:80-117, parse-bound:
// ~0.1 GB/s) and writes assignments as text (io.cpp:274-283).  Here records
// are raw float32 behind a 64-byte header and stream straight into pinned
// buffers: a reader thread pread()s chunk c+1 while chunk c is copied to the
// device, classified by st_eval_device and its labels copied back -- the file
// never has to fit in host memory.  u8 label files are narrowed on the
// device (k_narrow_u8) so a 10^9-record run writes 1 GB instead of 4 GB.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/spectree_b200.h"

namespace st_internal {
void set_error(const std::string& msg);
void set_launches(uint32_t n);
}  // namespace st_internal

namespace {

constexpr char kRecMagic[8] = {'S', 'T', 'R', 'E', 'C', '0', '0', '1'};
constexpr char kLabMagic[8] = {'S', 'T', 'L', 'A', 'B', '0', '0', '1'};
constexpr uint32_t kRecHeader = 64;
constexpr uint32_t kLabHeader = 32;

struct IoFail {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, std::string msg) { throw IoFail{code, std::move(msg)}; }

template <class F>
int guarded(F&& f) {
  try {
    f();
    st_internal::set_error("");
    return ST_OK;
  } catch (const IoFail& e) {
    st_internal::set_error(e.msg);
    return e.code;
  } catch (const std::bad_alloc&) {
    st_internal::set_error("host allocation failed");
    return ST_ERR_CUDA;
  } catch (const std::exception& e) {
    st_internal::set_error(e.what());
    return ST_ERR_IO;
  }
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? ST_ERR_NO_DEVICE : ST_ERR_CUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

void pread_all(int fd, void* dst, uint64_t bytes, uint64_t off, const std::string& path) {
  auto* p = static_cast<char*>(dst);
  while (bytes) {
    const ssize_t r = ::pread(fd, p, std::min<uint64_t>(bytes, 1ull << 30), (off_t)off);
    if (r <= 0) fail(ST_ERR_IO, path + ": short read at byte " + std::to_string(off));
    p += r;
    off += (uint64_t)r;
    bytes -= (uint64_t)r;
  }
}

void write_all(std::FILE* f, const void* src, uint64_t bytes, const std::string& path) {
  if (bytes && std::fwrite(src, 1, bytes, f) != bytes) fail(ST_ERR_IO, "cannot write " + path);
}

struct Fnv {  // dataset_checksum (dataset.cpp:76-93)
  uint64_t h = 0xcbf29ce484222325ull;
  void mix(const void* d, uint64_t n) {
    const auto* p = static_cast<const unsigned char*>(d);
    for (uint64_t i = 0; i < n; ++i) {
      h ^= p[i];
      h *= 0x100000001b3ull;
    }
  }
};

st_dataset_info read_info(int fd, const std::string& path) {
  unsigned char hd[kRecHeader];
  pread_all(fd, hd, kRecHeader, 0, path);
  if (std::memcmp(hd, kRecMagic, 8) != 0) fail(ST_ERR_IO, path + ": not a STREC001 record file");
  uint32_t version, layout, arity, flags;
  uint64_t count, sum;
  std::memcpy(&version, hd + 8, 4);
  std::memcpy(&layout, hd + 12, 4);
  std::memcpy(&count, hd + 16, 8);
  std::memcpy(&arity, hd + 24, 4);
  std::memcpy(&flags, hd + 28, 4);
  std::memcpy(&sum, hd + 32, 8);
  if (version != 1) fail(ST_ERR_IO, path + ": unsupported record file version " + std::to_string(version));
  if (layout != ST_LAYOUT_AOS && layout != ST_LAYOUT_SOA)
    fail(ST_ERR_IO, path + ": bad layout " + std::to_string(layout));
  if (arity == 0) fail(ST_ERR_IO, path + ": dataset arity must be >= 1");
  const off_t end = ::lseek(fd, 0, SEEK_END);
  // count * arity * 4 must not wrap: a crafted header could otherwise pass
  // the size check on a short file and size the caller's allocations
  if (count > (UINT64_MAX - kRecHeader) / (4ull * arity) || end < 0 ||
      (uint64_t)end != kRecHeader + count * (uint64_t)arity * 4)
    fail(ST_ERR_IO, path + ": file size does not match " + std::to_string(count) + " records of arity " +
                        std::to_string(arity));
  st_dataset_info in{};
  in.count = count;
  in.arity = arity;
  in.layout = layout;
  in.has_checksum = flags & 1u;
  in.checksum = sum;
  in.data_offset = kRecHeader;
  return in;
}

int open_read(const std::string& path) {
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) fail(ST_ERR_IO, "cannot open " + path + " for reading");
  return fd;
}

// Records [first, first+n) as AoS into out (n*arity floats).
void read_rows(int fd, const st_dataset_info& in, uint64_t first, uint64_t n, float* out,
               std::vector<float>& scratch, const std::string& path) {
  const uint64_t a = in.arity;
  if (in.layout == ST_LAYOUT_AOS) {
    pread_all(fd, out, n * a * 4, in.data_offset + first * a * 4, path);
    return;
  }
  scratch.resize(n);
  for (uint64_t k = 0; k < a; ++k) {
    pread_all(fd, scratch.data(), n * 4, in.data_offset + (k * in.count + first) * 4, path);
    for (uint64_t r = 0; r < n; ++r) out[r * a + k] = scratch[r];
  }
}

uint64_t file_checksum(int fd, const st_dataset_info& in, const std::string& path) {
  Fnv f;
  const uint32_t a = in.arity;
  const uint64_t m = in.count;
  f.mix(&a, 4);
  f.mix(&m, 8);
  const uint64_t rows = std::max<uint64_t>(1, (16ull << 20) / (4ull * a));
  std::vector<float> buf, scratch;
  for (uint64_t r = 0; r < m; r += rows) {
    const uint64_t n = std::min(rows, m - r);
    buf.resize(n * a);
    read_rows(fd, in, r, n, buf.data(), scratch, path);
    f.mix(buf.data(), n * a * 4);
  }
  return f.h;
}

__global__ void k_narrow_u8(const uint32_t* __restrict__ in, uint8_t* __restrict__ out, uint64_t n) {
  // 4 labels -> one 32-bit store per thread (grid-stride, coalesced)
  const uint64_t q = (n + 3) / 4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < q; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = 4 * i;
    if (b + 4 <= n) {
      const uint4 v = *reinterpret_cast<const uint4*>(in + b);
      *reinterpret_cast<uint32_t*>(out + b) = (v.x & 0xFF) | (v.y & 0xFF) << 8 | (v.z & 0xFF) << 16 | (v.w & 0xFF) << 24;
    } else {
      for (uint64_t k = b; k < n; ++k) out[k] = (uint8_t)in[k];
    }
  }
}

}  // namespace

extern "C" {

int st_dataset_save(const char* path, const float* x, uint64_t m, uint32_t a, int layout,
                    int with_checksum) {
  return guarded([&] {
    if (!path) fail(ST_ERR_ARGUMENT, "null path");
    if (a == 0) fail(ST_ERR_ARGUMENT, "dataset arity must be >= 1");
    if (layout != ST_LAYOUT_AOS && layout != ST_LAYOUT_SOA) fail(ST_ERR_ARGUMENT, "bad layout");
    if (m && !x) fail(ST_ERR_ARGUMENT, "null records");
    uint64_t sum = 0;
    if (with_checksum) {
      Fnv f;
      f.mix(&a, 4);
      f.mix(&m, 8);
      if (layout == ST_LAYOUT_AOS) {
        f.mix(x, m * a * 4ull);
      } else {
        std::vector<float> row(a);
        for (uint64_t r = 0; r < m; ++r) {
          for (uint32_t k = 0; k < a; ++k) row[k] = x[k * m + r];
          f.mix(row.data(), a * 4ull);
        }
      }
      sum = f.h;
    }
    std::FILE* fp = std::fopen(path, "wb");
    if (!fp) fail(ST_ERR_IO, std::string("cannot open ") + path + " for writing");
    struct Close {
      std::FILE* f;
      ~Close() {
        if (f) std::fclose(f);
      }
    } guard{fp};
    unsigned char hd[kRecHeader] = {};
    const uint32_t version = 1, lay = (uint32_t)layout, flags = with_checksum ? 1u : 0u;
    std::memcpy(hd, kRecMagic, 8);
    std::memcpy(hd + 8, &version, 4);
    std::memcpy(hd + 12, &lay, 4);
    std::memcpy(hd + 16, &m, 8);
    std::memcpy(hd + 24, &a, 4);
    std::memcpy(hd + 28, &flags, 4);
    std::memcpy(hd + 32, &sum, 8);
    write_all(fp, hd, kRecHeader, path);
    write_all(fp, x, m * a * 4ull, path);
    guard.f = nullptr;
    if (std::fclose(fp) != 0) fail(ST_ERR_IO, std::string("cannot write ") + path);
  });
}

int st_dataset_info_read(const char* path, st_dataset_info* out) {
  return guarded([&] {
    if (!path || !out) fail(ST_ERR_ARGUMENT, "null argument");
    Fd fd{open_read(path)};
    *out = read_info(fd.fd, path);
  });
}

int st_dataset_load(const char* path, uint64_t first, uint64_t count, float* out, int verify) {
  return guarded([&] {
    if (!path) fail(ST_ERR_ARGUMENT, "null path");
    Fd fd{open_read(path)};
    const st_dataset_info in = read_info(fd.fd, path);
    if (first > in.count || count > in.count - first)
      fail(ST_ERR_ARGUMENT, "record range [" + std::to_string(first) + ", " + std::to_string(first + count) +
                                ") outside the file's " + std::to_string(in.count) + " records");
    if (count && !out) fail(ST_ERR_ARGUMENT, "null output");
    if (verify) {
      if (!in.has_checksum) fail(ST_ERR_IO, std::string(path) + ": no checksum to verify");
      if (file_checksum(fd.fd, in, path) != in.checksum)
        fail(ST_ERR_IO, std::string(path) + ": dataset checksum mismatch");
    }
    std::vector<float> scratch;
    read_rows(fd.fd, in, first, count, out, scratch, path);
  });
}

int st_labels_save(const char* path, const uint32_t* labels, uint64_t m, uint32_t width) {
  return guarded([&] {
    if (!path) fail(ST_ERR_ARGUMENT, "null path");
    if (width != 1 && width != 4) fail(ST_ERR_ARGUMENT, "label width must be 1 or 4");
    if (m && !labels) fail(ST_ERR_ARGUMENT, "null labels");
    std::vector<uint8_t> narrow;
    if (width == 1) {
      narrow.resize(m);
      for (uint64_t i = 0; i < m; ++i) {
        if (labels[i] > 255) fail(ST_ERR_ARGUMENT, "class " + std::to_string(labels[i]) + " does not fit in u8");
        narrow[i] = (uint8_t)labels[i];
      }
    }
    std::FILE* fp = std::fopen(path, "wb");
    if (!fp) fail(ST_ERR_IO, std::string("cannot open ") + path + " for writing");
    unsigned char hd[kLabHeader] = {};
    const uint32_t version = 1;
    std::memcpy(hd, kLabMagic, 8);
    std::memcpy(hd + 8, &version, 4);
    std::memcpy(hd + 12, &width, 4);
    std::memcpy(hd + 16, &m, 8);
    bool ok = std::fwrite(hd, 1, kLabHeader, fp) == kLabHeader;
    if (width == 1) ok = ok && (m == 0 || std::fwrite(narrow.data(), 1, m, fp) == m);
    else ok = ok && (m == 0 || std::fwrite(labels, 4, m, fp) == m);
    ok = (std::fclose(fp) == 0) && ok;
    if (!ok) fail(ST_ERR_IO, std::string("cannot write ") + path);
  });
}

int st_labels_load(const char* path, uint32_t* out, uint64_t cap, uint64_t* count, uint32_t* width) {
  return guarded([&] {
    if (!path) fail(ST_ERR_ARGUMENT, "null path");
    Fd fd{open_read(path)};
    unsigned char hd[kLabHeader];
    pread_all(fd.fd, hd, kLabHeader, 0, path);
    if (std::memcmp(hd, kLabMagic, 8) != 0) fail(ST_ERR_IO, std::string(path) + ": not a STLAB001 label file");
    uint32_t version, w;
    uint64_t m;
    std::memcpy(&version, hd + 8, 4);
    std::memcpy(&w, hd + 12, 4);
    std::memcpy(&m, hd + 16, 8);
    if (version != 1 || (w != 1 && w != 4)) fail(ST_ERR_IO, std::string(path) + ": bad label header");
    const off_t end = ::lseek(fd.fd, 0, SEEK_END);
    if (m > (UINT64_MAX - kLabHeader) / w || end < 0 || (uint64_t)end != kLabHeader + m * w)
      fail(ST_ERR_IO, std::string(path) + ": truncated label file");
    if (count) *count = m;
    if (width) *width = w;
    if (!out) return;
    if (cap < m) fail(ST_ERR_ARGUMENT, "label buffer too small");
    if (w == 4) {
      pread_all(fd.fd, out, m * 4, kLabHeader, path);
    } else {
      std::vector<uint8_t> b(m);
      pread_all(fd.fd, b.data(), m, kLabHeader, path);
      for (uint64_t i = 0; i < m; ++i) out[i] = b[i];
    }
  });
}

int st_eval_file(const st_tree* tree, const char* data_path, const st_geom* geom,
                 const char* labels_path, uint32_t width, uint64_t* records_out) {
  return guarded([&] {
    if (!tree || !data_path || !labels_path) fail(ST_ERR_ARGUMENT, "null argument");
    if (width != 1 && width != 4) fail(ST_ERR_ARGUMENT, "label width must be 1 or 4");
    st_tree_info ti{};
    if (int rc = st_tree_get_info(tree, &ti)) throw IoFail{rc, "tree info failed"};
    if (width == 1 && ti.max_class > 255)
      fail(ST_ERR_ARGUMENT, "u8 labels need every class < 256 (tree has class " + std::to_string(ti.max_class) + ")");
    Fd fd{open_read(data_path)};
    const st_dataset_info in = read_info(fd.fd, data_path);
    if (ti.max_attribute >= in.arity)  // check_attribute_range (eval_serial.cpp:10-17), before any work
      fail(ST_ERR_ARGUMENT, "tree reads attribute " + std::to_string(ti.max_attribute) +
                                " but records have arity " + std::to_string(in.arity));
    std::FILE* fo = std::fopen(labels_path, "wb");
    if (!fo) fail(ST_ERR_IO, std::string("cannot open ") + labels_path + " for writing");
    struct Close {
      std::FILE* f;
      ~Close() {
        if (f) std::fclose(f);
      }
    } oguard{fo};
    {
      unsigned char hd[kLabHeader] = {};
      const uint32_t version = 1;
      std::memcpy(hd, kLabMagic, 8);
      std::memcpy(hd + 8, &version, 4);
      std::memcpy(hd + 12, &width, 4);
      std::memcpy(hd + 16, &in.count, 8);
      write_all(fo, hd, kLabHeader, labels_path);
    }
    const uint64_t m = in.count, a = in.arity;
    uint64_t launches = 0;
    if (m > 0) {
      int count = 0;
      if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        fail(ST_ERR_NO_DEVICE, "no CUDA device available (no CPU fallback)");
      }
      constexpr int kBufs = 3;
      const uint64_t chunk = std::min<uint64_t>(m, std::max<uint64_t>(1024, ((64ull << 20) / (4 * a)) / 1024 * 1024));
      const uint64_t n_chunks = (m + chunk - 1) / chunk;
      struct Buf {
        float* host = nullptr;
        float* dev = nullptr;
        uint32_t* dlab = nullptr;
        uint8_t* dlab8 = nullptr;
        void* hlab = nullptr;
        cudaStream_t s = nullptr;
        cudaEvent_t done = nullptr;
      };
      std::vector<Buf> b(kBufs);
      struct Release {
        std::vector<Buf>& b;
        ~Release() {
          for (Buf& x : b) {
            if (x.s) cudaStreamSynchronize(x.s);
            cudaFreeHost(x.host);
            cudaFreeHost(x.hlab);
            cudaFree(x.dev);
            cudaFree(x.dlab);
            cudaFree(x.dlab8);
            if (x.done) cudaEventDestroy(x.done);
            if (x.s) cudaStreamDestroy(x.s);
          }
        }
      } release{b};
      for (Buf& x : b) {
        ck(cudaMallocHost(&x.host, chunk * a * 4), "cudaMallocHost(records)");
        ck(cudaMallocHost(&x.hlab, chunk * 4), "cudaMallocHost(labels)");
        ck(cudaMalloc(&x.dev, chunk * a * 4), "cudaMalloc(records)");
        ck(cudaMalloc(&x.dlab, chunk * 4), "cudaMalloc(labels)");
        if (width == 1) ck(cudaMalloc(&x.dlab8, chunk), "cudaMalloc(u8 labels)");
        ck(cudaStreamCreateWithFlags(&x.s, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming), "cudaEventCreate");
      }
      // Reader thread: fills host buffer c % kBufs with chunk c once the
      // consumer has released it (its H2D finished).
      std::mutex mu;
      std::condition_variable cv;
      std::vector<int> filled(kBufs, -1);      // chunk index held by each buffer, -1 = empty
      std::vector<bool> free_slot(kBufs, true);
      std::string reader_err;
      bool abort = false;
      std::thread reader([&] {
        std::vector<float> scratch;
        try {
          for (uint64_t c = 0; c < n_chunks; ++c) {
            const int k = (int)(c % kBufs);
            {
              std::unique_lock<std::mutex> lk(mu);
              cv.wait(lk, [&] { return free_slot[k] || abort; });
              if (abort) return;
              free_slot[k] = false;
            }
            const uint64_t r0 = c * chunk, n = std::min(chunk, m - r0);
            read_rows(fd.fd, in, r0, n, b[k].host, scratch, data_path);
            {
              std::lock_guard<std::mutex> lk(mu);
              filled[k] = (int)c;
            }
            cv.notify_all();
          }
        } catch (const IoFail& e) {
          std::lock_guard<std::mutex> lk(mu);
          reader_err = e.msg;
          abort = true;
          cv.notify_all();
        }
      });
      struct Join {
        std::thread& t;
        std::mutex& mu;
        std::condition_variable& cv;
        bool& abort;
        ~Join() {
          {
            std::lock_guard<std::mutex> lk(mu);
            abort = true;
          }
          cv.notify_all();
          if (t.joinable()) t.join();
        }
      } join{reader, mu, cv, abort};
      // chunks whose labels are in flight, in file order
      std::vector<uint64_t> pending;
      auto retire = [&](uint64_t c) {
        const int k = (int)(c % kBufs);
        ck(cudaEventSynchronize(b[k].done), "label copy");
        const uint64_t n = std::min(chunk, m - c * chunk);
        write_all(fo, b[k].hlab, n * width, labels_path);
      };
      for (uint64_t c = 0; c < n_chunks; ++c) {
        const int k = (int)(c % kBufs);
        if (c >= (uint64_t)kBufs) retire(c - kBufs);  // buffer k's previous chunk
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return filled[k] == (int)c || abort; });
          if (filled[k] != (int)c) fail(ST_ERR_IO, reader_err.empty() ? "reader aborted" : reader_err);
        }
        const uint64_t n = std::min(chunk, m - c * chunk);
        Buf& x = b[k];
        ck(cudaMemcpyAsync(x.dev, x.host, n * a * 4, cudaMemcpyHostToDevice, x.s), "H2D");
        // the host buffer is reusable once the copy has been consumed
        ck(cudaStreamSynchronize(x.s), "H2D");
        {
          std::lock_guard<std::mutex> lk(mu);
          filled[k] = -1;
          free_slot[k] = true;
        }
        cv.notify_all();
        if (int rc = st_eval_device(tree, x.dev, n, (uint32_t)a, 0, ST_LAYOUT_AOS, geom, x.dlab, nullptr, x.s))
          throw IoFail{rc, std::string("chunk ") + std::to_string(c) + ": " + st_last_error()};
        launches += st_last_launch_count();
        if (width == 1) {
          k_narrow_u8<<<(unsigned)std::min<uint64_t>(1184, (n / 4 + 255) / 256 + 1), 256, 0, x.s>>>(x.dlab, x.dlab8, n);
          ck(cudaGetLastError(), "narrow kernel launch");
          ++launches;
          ck(cudaMemcpyAsync(x.hlab, x.dlab8, n, cudaMemcpyDeviceToHost, x.s), "D2H");
        } else {
          ck(cudaMemcpyAsync(x.hlab, x.dlab, n * 4, cudaMemcpyDeviceToHost, x.s), "D2H");
        }
        ck(cudaEventRecord(x.done, x.s), "event");
      }
      for (uint64_t c = n_chunks > (uint64_t)kBufs ? n_chunks - kBufs : 0; c < n_chunks; ++c) retire(c);
    }
    oguard.f = nullptr;
    if (std::fclose(fo) != 0) fail(ST_ERR_IO, std::string("cannot write ") + labels_path);
    if (records_out) *records_out = m;
    st_internal::set_launches((uint32_t)std::min<uint64_t>(launches, 0xFFFFFFFFu));
  });
}

}  // extern "C"

// Probe for an attribute-group "plane" record tile (16-attribute records):
// can TMA stage a tile as 4 planes of [R records][4 attributes] (a 3D box
// {4, R, 4} over dims {4 attrs, m records, 4 groups} with strides {64, 16} B)
// as fast as the record-major 2D box, and how many shared-memory cycles do
// random feature reads cost in each layout?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_plane_probe tma_plane_probe.cu && ./tma_plane_probe
//
// Modes: 0 = record-major 2D box with SWIZZLE_128B (the data kernel's tile),
//        1 = planes of 4 attributes (3D box {4, R, 4}), 2 = planes of 8 ({8, R, 2}).  Each warp streams 128-record tiles
// through a one-stage ring (TMA, mbarrier) and does `reads` rounds of one
// random attribute read per lane per record chain (4 chains), like a walk's
// feature loads.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      std::printf("%s: %s\n", #x, cudaGetErrorString(e));                             \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

constexpr int R = 128, A = 16, WARPS = 24;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(WARPS * 32) k_probe(const __grid_constant__ CUtensorMap tmap, int mode, uint64_t m,
                                                      int reads, uint32_t* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = (smem_u32(smem) + 1023u) & ~1023u;
  const uint32_t tile = base + warp * (R * A * 4);
  const uint32_t bar = base + WARPS * (R * A * 4) + 8 * warp;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const uint64_t n_tiles = m / R;
  uint32_t acc = 0, phase = 0;
  for (uint64_t t = (uint64_t)blockIdx.x * WARPS + warp; t < n_tiles; t += (uint64_t)gridDim.x * WARPS) {
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(R * A * 4) : "memory");
      if (mode == 0)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                tile),
            "l"(&tmap), "r"(0), "r"((int)(t * R * A / 32)), "r"(bar)
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                tile),
            "l"(&tmap), "r"(0), "r"((int)(t * R)), "r"(0), "r"(bar)
            : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(bar),
        "r"(phase)
        : "memory");
    phase ^= 1u;
    // 4 record chains per lane (records lane + 32 q), `reads` random feature reads each
    uint32_t h = (uint32_t)t * 2654435761u + lane * 40503u;
#pragma unroll 1
    for (int k = 0; k < reads; ++k) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        h = h * 1664525u + 1013904223u;
        const uint32_t a = h >> 28, r = lane + 32u * q;
        uint32_t addr;
        if (mode == 0) {
          const uint32_t f = (r * A + a) * 4u;
          addr = tile + (f ^ ((f >> 3) & 0x70u));
        } else if (mode == 1) {
          addr = tile + (a >> 2) * (R * 16u) + r * 16u + (a & 3u) * 4u;
        } else {
          addr = tile + (a >> 3) * (R * 32u) + r * 32u + (a & 7u) * 4u;
        }
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
        acc += v;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
  }
  if (acc == 0x12345678u) out[0] = acc;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const uint64_t m = 16ull << 20;  // 16M records x 64 B = 1 GiB
  float* x = nullptr;
  uint32_t* out = nullptr;
  CK(cudaMalloc(&x, m * A * 4));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(x, 0, m * A * 4));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  EncodeFn enc = (EncodeFn)p;
  CUtensorMap maps[3];
  {
    const cuuint64_t dims[2] = {32, m * A / 32};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {32, R * A / 32};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&maps[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
      std::printf("encode 2d failed\n");
  }
  {
    const cuuint64_t dims[3] = {4, m, 4};
    const cuuint64_t strides[2] = {64, 16};
    const cuuint32_t box[3] = {4, R, 4};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&maps[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) std::printf("encode 3d failed (%d)\n", (int)r);
  }
  {
    const cuuint64_t dims[3] = {8, m, 2};
    const cuuint64_t strides[2] = {64, 32};
    const cuuint32_t box[3] = {8, R, 2};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&maps[2], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) std::printf("encode 3d/8 failed (%d)\n", (int)r);
  }
  const size_t smem = 1024 + WARPS * (R * A * 4) + 8 * WARPS;
  CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int reads : {0, 12, 24}) {
    for (int mode : {0, 1, 2}) {
      for (int w = 0; w < 2; ++w) k_probe<<<sms, WARPS * 32, smem>>>(maps[mode], mode, m, reads, out);
      CK(cudaDeviceSynchronize());
      float best = 1e9f;
      for (int it = 0; it < 5; ++it) {
        cudaEventRecord(e0);
        k_probe<<<sms, WARPS * 32, smem>>>(maps[mode], mode, m, reads, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      std::printf("reads/record %2d  %-13s %.3f ms  %.0f GB/s\n", reads, mode == 2 ? "planes-8(3D)" : mode ? "planes-4(3D)" : "record-major", best,
                  m * A * 4 / (best * 1e-3) / 1e9);
    }
  }
  return 0;
}

// Shared-memory / shuffle / vote pipe throughput probe (sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mio_probe mio_probe.cu && ./mio_probe
// Per kernel: SM-cycles per warp-instruction at full occupancy (32 warps/SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 2048, kUnroll = 8, kWarps = 32;

template <int MODE>
__global__ void __launch_bounds__(1024) probe(uint32_t* out, uint32_t salt, uint32_t zero) {
  __shared__ __align__(16) uint32_t sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * 2654435761u;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, base = (uint32_t)__cvta_generic_to_shared(sm);
  uint32_t acc = salt;
  uint32_t addr;
  // MODE 0: LDS.128, lanes 4g..4g+3 read the same 16 B, 8 groups on 8 distinct bank quads
  // MODE 1: LDS.64, 32 lanes x 8 B consecutive (256 B)
  // MODE 2: LDS.32, 32 lanes x 4 B consecutive (128 B)
  // MODE 3: LDS.32, lanes 4g..4g+3 same word, 8 groups distinct banks
  // MODE 4: SHFL.IDX width 4
  // MODE 5: VOTE.BALLOT
  // MODE 6: LDS.128, 8 groups x 16 B, each group own chunk, groups 2-way on quads (conflict)
  // MODE 7: LDS.64, lanes 4g+j read chunk g word pair j (32 B per group)
  if (MODE == 0) addr = base + 16u * (lane >> 2);
  else if (MODE == 1 || MODE == 7) addr = base + 8u * lane;
  else if (MODE == 2) addr = base + 4u * lane;
  else if (MODE == 3) addr = base + 4u * (lane >> 2);
  else if (MODE == 8) addr = base + 8u * (lane >> 2);
  else if (MODE >= 9) addr = base + 4u * lane;
  else if (MODE == 6) addr = base + 16u * ((lane >> 2) & 3) + 256u * (lane >> 4);
  else addr = base;
#pragma unroll 1
  for (int it = 0; it < kIters; ++it) {
    const uint32_t addr_it = addr ^ (it * zero);  // zero at run time: defeats hoisting
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t addr = addr_it + u * (zero << 4);
      if (MODE == 0 || MODE == 6) {
        uint32_t a, b, c, d;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr) : "memory");
        acc ^= a + b + c + d;
      } else if (MODE == 1 || MODE == 7) {
        uint32_t a, b;
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(addr) : "memory");
        acc ^= a + b;
      } else if (MODE == 2 || MODE == 3) {
        uint32_t a;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a) : "r"(addr) : "memory");
        acc ^= a;
      } else if (MODE == 4) {
        uint32_t v;
        asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1c1f, 0xffffffff;" : "=r"(v) : "r"(acc + u), "r"(lane + u + addr) : "memory");
        acc ^= v;
      } else if (MODE == 8) {
        uint32_t a, b;
        asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(addr) : "memory");
        acc ^= a + b;
      } else if (MODE == 9 || MODE == 10 || MODE == 11) {
        uint32_t a, v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a) : "r"(addr) : "memory");
        if (MODE == 9)
          asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; vote.sync.ballot.b32 %0, p, 0xffffffff;}" : "=r"(v) : "r"(acc & (1u << u)) : "memory");
        else if (MODE == 10)
          asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1c1f, 0xffffffff;" : "=r"(v) : "r"(acc + u), "r"(lane + u + addr) : "memory");
        else
          asm volatile("redux.sync.or.b32 %0, %1, 0xffffffff;" : "=r"(v) : "r"((acc & 1u) << lane) : "memory");
        acc ^= a + v;
      } else if (MODE == 12 || MODE == 13 || MODE == 14 || MODE == 15) {
        uint32_t v;
        if (MODE == 12)  // full-width idx, computed source lane
          asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(v) : "r"(acc + u), "r"((lane & ~3u) | ((lane + u + addr) & 3u)) : "memory");
        else if (MODE == 13)
          asm volatile("shfl.sync.bfly.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(v) : "r"(acc + u), "r"((u + addr) & 31u) : "memory");
        else if (MODE == 14)  // width 4 but uniform source index
          asm volatile("shfl.sync.idx.b32 %0, %1, 0, 0x1c1f, 0xffffffff;" : "=r"(v) : "r"(acc + u + addr) : "memory");
        else  // full-width idx, all lanes read lane 0
          asm volatile("shfl.sync.idx.b32 %0, %1, 0, 0x1f, 0xffffffff;" : "=r"(v) : "r"(acc + u + addr) : "memory");
        acc ^= v;
      } else if (MODE == 5) {
        { uint32_t v; asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; vote.sync.ballot.b32 %0, p, 0xffffffff;}" : "=r"(v) : "r"(acc & (1u << u)) : "memory"); acc += v; }
      }
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE>
float run(int sms) {
  uint32_t* out;
  cudaMalloc(&out, 4);
  probe<MODE><<<sms * 2, kWarps * 16>>>(out, 1, 0);  // warm
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  probe<MODE><<<sms * 2, kWarps * 16>>>(out, 1, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double warp_instr_per_sm = (double)kWarps * kIters * kUnroll;
  const double cycles = ms * 1e-3 * khz * 1e3;
  cudaFree(out);
  return (float)(cycles / warp_instr_per_sm);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"LDS.128 bcast 8 chunks", "LDS.64 256B contiguous", "LDS.32 128B contiguous",
                         "LDS.32 bcast 8 words", "SHFL.IDX w4", "VOTE.BALLOT", "LDS.128 bcast 2-way quad",
                         "LDS.64 (same as 1)", "LDS.64 bcast 8 words", "LDS.32 + VOTE (pair)", "LDS.32 + SHFL (pair)",
                         "LDS.32 + REDUX.OR (pair)", "SHFL.IDX w32 computed src", "SHFL.BFLY", "SHFL.IDX w4 src 0",
                         "SHFL.IDX w32 src 0"};
  float r[16] = {run<0>(sms), run<1>(sms), run<2>(sms), run<3>(sms), run<4>(sms), run<5>(sms),
                 run<6>(sms), run<7>(sms), run<8>(sms), run<9>(sms), run<10>(sms), run<11>(sms),
                 run<12>(sms), run<13>(sms), run<14>(sms), run<15>(sms)};
  for (int i = 0; i < 16; ++i) printf("%-28s %.3f SM-cycles per warp-instruction (at max clock)\n", names[i], r[i]);
  return 0;
}

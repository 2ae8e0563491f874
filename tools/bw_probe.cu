// Bandwidth probe for the column-tile staging structure of pipe_body
// (kernel_common.cuh): one TMA producer warp + W consumer warps per CTA,
// `stages` tiles of `tile` rows x 7 columns (88 B/row, the Q1 scan) in a ring.
// Consumers do almost nothing (xor of one word per row) so the number is the
// ceiling the staging structure reaches on this GPU; a plain LDG.128
// grid-stride read of the same bytes is printed beside it.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bw_probe tools/bw_probe.cu
//   tools/bw_probe
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef unsigned long long u64;
typedef unsigned int u32;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, u32 c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, u32 par) {
  u32 ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok)
                 : "r"(smem_u32(b)), "r"(par)
                 : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, u32 bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

struct Cols {
  const uint8_t* p[7];
  u32 w[7];
};

template <int W>
__global__ void __launch_bounds__((W + 1) * 32, 1) staged(Cols c, u64 rows, u32 tile, u32 stages, u64* sink, u32 work) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 8;
  uint8_t* ring = sm + 128;
  const u32 stage_bytes = tile * 88;
  const u32 ntiles = (u32)(rows / tile);
  const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (u32 s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == W) {
    if (lane == 0) {
      u32 s = 0, ph = 0, k = 0;
      for (u32 t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        if (k >= stages) mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = ring + s * stage_bytes;
        mbar_expect(&full[s], stage_bytes);
        u32 off = 0;
        for (int i = 0; i < 7; ++i) {
          bulk(st + off, c.p[i] + (u64)t * tile * c.w[i], tile * c.w[i], &full[s]);
          off += tile * c.w[i];
        }
        if (++s == stages) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  u64 acc = 0;
  u32 s = 0, ph = 0;
  for (u32 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(&full[s], ph);
    const uint8_t* st = ring + s * stage_bytes;
    for (u32 r = warp * 32 + lane; r < tile; r += W * 32) acc ^= ((const u64*)st)[r];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    // synthetic per-tile compute after the release (models the aggregation work)
    u64 x = acc | 1;
    for (u32 i = 0; i < work; ++i) x = x * 0x9E3779B97F4A7C15ull + i;
    acc ^= x;
    if (++s == stages) { s = 0; ph ^= 1; }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

__global__ void plain(const ulonglong2* p, u64 n16, u64* sink) {
  ulonglong2 a = {0, 0};
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x, st = (u64)gridDim.x * blockDim.x;
  for (; i + 3 * st < n16; i += 4 * st) {
    ulonglong2 x0 = p[i], x1 = p[i + st], x2 = p[i + 2 * st], x3 = p[i + 3 * st];
    a.x ^= x0.x ^ x1.x ^ x2.x ^ x3.x;
    a.y ^= x0.y ^ x1.y ^ x2.y ^ x3.y;
  }
  for (; i < n16; i += st) { a.x ^= p[i].x; a.y ^= p[i].y; }
  if ((a.x ^ a.y) == 0x1234567) sink[0] = a.x;
}

int main() {
  const u64 rows = 60000000ull / 2048 * 2048;
  const u32 w[7] = {8, 8, 8, 16, 16, 16, 16};
  Cols c;
  std::vector<void*> bufs;
  for (int i = 0; i < 7; ++i) {
    void* p;
    cudaMalloc(&p, rows * w[i]);
    cudaMemset(p, i, rows * w[i]);
    c.p[i] = (const uint8_t*)p;
    c.w[i] = w[i];
  }
  void* flush;
  const size_t fl = 512ull << 20;
  cudaMalloc(&flush, fl);
  u64* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = rows * 88.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    float best = 1e9, sum = 0;
    for (int it = 0; it < 8; ++it) {
      cudaMemsetAsync(flush, it, fl);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) { sum += ms; best = ms < best ? ms : best; }
    }
    return std::make_pair(best, sum / 6);
  };
  {
    u64 n16 = rows * 8 / 16;  // the 8-byte columns as one stream (rough)
    auto r = timeit([&] { plain<<<sms * 8, 256>>>((const ulonglong2*)c.p[3], rows * 16 / 16, sink); });
    printf("plain LDG.128 one 16B column: %.3f ms  %.0f GB/s\n", r.first, rows * 16.0 / r.first / 1e6);
    (void)n16;
  }
  u32 work = 0;
  auto run = [&](auto kern, int W, u32 tile, u32 stages, int cpsm) {
    size_t smem = 128 + (size_t)stages * tile * 88;
    if (smem > 227 * 1024) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, (W + 1) * 32, smem);
    if (occ < cpsm) return;
    auto r = timeit([&] { kern<<<sms * cpsm, (W + 1) * 32, smem>>>(c, rows, tile, stages, sink, work); });
    cudaError_t e = cudaGetLastError();
    printf("work=%4u W=%2d tile=%5u stages=%u ctas/sm=%d smem=%6zu  best %.3f ms avg %.3f ms  %.0f GB/s (avg %.0f) %s\n", W,
           work, tile, stages, cpsm, smem, r.first, r.second, bytes / r.first / 1e6, bytes / r.second / 1e6,
           e ? cudaGetErrorString(e) : "");
  };
  for (u32 wk : {0u, 40u, 80u, 120u, 160u}) {
    work = wk;
    for (u32 stages : {2u, 3u, 4u}) run(staged<16>, 16, 512, stages, 1);
    for (u32 stages : {4u, 6u, 8u}) run(staged<16>, 16, 256, stages, 1);
  }
  return 0;
}

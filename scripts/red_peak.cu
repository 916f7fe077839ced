// red_peak.cu -- measured peaks of the atomic reductions the build uses, for
// the "atomic throughput against B200 peak" evidence.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/red_peak scripts/red_peak.cu
//   /tmp/red_peak > profiles/red_peak.json
//
// Each case issues one atomicMax (uint32, result unused -> RED) per element
// of a stream of pseudo-random addresses and is timed with CUDA events (best
// of 5 after a warm-up):
//   global_l2    keys in a 64 MiB buffer (L2-resident: the cfg1 atomic build's
//                108 MB of keys are about this size)
//   global_dram  keys in a 4 GiB buffer (the cfg3 key planes would be 5.6 GB:
//                every RED a DRAM read-modify-write)
//   global_warp_uniform  all lanes of a warp on one address (CREDUX + one RED)
//   shared       per-CTA 48 KiB table (the partitioned builds' reductions)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__global__ void red_global(uint32_t *keys, uint32_t mask, int64_t n, int uniform) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t h = hash32((uint32_t)(uniform ? (i >> 5) : i));
    atomicMax(keys + (h & mask), (uint32_t)i);
  }
}

__global__ void red_shared(uint32_t *out, int64_t n) {
  __shared__ uint32_t tab[12288];
  for (int t = threadIdx.x; t < 12288; t += blockDim.x) tab[t] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    atomicMax(tab + hash32((uint32_t)i) % 12288u, (uint32_t)i);
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = tab[blockIdx.x % 12288];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t big = (size_t)4 << 30;
  uint32_t *keys = nullptr;
  if (cudaMalloc(&keys, big) != cudaSuccess) return 1;
  cudaMemset(keys, 0, big);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int64_t n = (int64_t)1 << 30;  // operations per case
  auto time = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    return best;
  };
  const int grid = sms * 8, block = 256;
  const float t_l2 = time([&] { red_global<<<grid, block>>>(keys, (16u << 20) - 1u, n, 0); });
  const float t_dram = time([&] { red_global<<<grid, block>>>(keys, (1u << 30) - 1u, n, 0); });
  const float t_uni = time([&] { red_global<<<grid, block>>>(keys, (1u << 30) - 1u, n, 1); });
  const float t_sh = time([&] { red_shared<<<sms * 4, 512>>>(keys, n * 4); });
  const cudaError_t e = cudaGetLastError();
  printf("{\"ops_per_case\": %lld, \"sms\": %d, \"error\": \"%s\",\n", (long long)n, sms,
         cudaGetErrorString(e));
  printf(" \"global_l2_red_gops\": %.1f,\n", n / (t_l2 * 1e6));
  printf(" \"global_dram_red_gops\": %.1f,\n", n / (t_dram * 1e6));
  printf(" \"global_warp_uniform_gops\": %.1f,\n", n / (t_uni * 1e6));
  printf(" \"shared_atom_gops\": %.1f,\n", 4 * n / (t_sh * 1e6));
  printf(" \"how\": \"atomicMax uint32 at hashed addresses, result unused (RED), best of 5, CUDA events\"}\n");
  cudaFree(keys);
  return 0;
}

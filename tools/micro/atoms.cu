// microbenchmark: shared-memory atomicOr throughput vs same-address lanes per instruction
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(unsigned* out, int iters, int group) {
  __shared__ unsigned s[8][1024];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = lane; i < 1024; i += 32) s[w][i] = 0;
  __syncwarp();
  unsigned x = (blockIdx.x * 8 + w) * 2654435761u;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    const unsigned base = (x >> 20) & 1023u;
    const unsigned a = (base + lane / group * 33) & 1023u;   // `group` lanes share an address
    if (MODE == 0) atomicOr(&s[w][a], 1u << (lane & 31));
    else if (MODE == 1) { s[w][a] |= 1u << (lane & 31); }
    else { unsigned v = s[w][a]; x ^= v; }
  }
  __syncwarp();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s[w][lane] ^ x;
}
int main() {
  unsigned* out; cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int group : {1, 2, 3, 4, 8, 32}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<148 * 8, 256>>>(out, iters, group);
        else if (mode == 1) k<1><<<148 * 8, 256>>>(out, iters, group);
        else k<2><<<148 * 8, 256>>>(out, iters, group);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double warp_ops = 148.0 * 8 * 8 * iters;
        if (rep) printf("mode %s group %2d: %.3f ms, %.2f warp-ops/clk/SM (at 1.9 GHz)\n",
                        mode == 0 ? "ATOMS.OR" : mode == 1 ? "LDS+STS " : "LDS     ", group, ms,
                        warp_ops / (ms * 1e-3) / 148 / 1.9e9);
      }
    }
  return 0;
}

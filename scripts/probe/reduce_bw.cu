// Probe: bandwidth of the W-slot ReduceScatter reduction pattern
// (out = sum of W bf16 slots, fp32 accumulate) as a function of the slot
// stride (exactly rows*n*2 = 16 MB at C4/TP=8, or padded) and of how many
// loads a thread keeps in flight.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/reduce_bw scripts/probe/reduce_bw.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>

template <int W, int ROWS>
__global__ void __launch_bounds__(256) red(const uint4* __restrict__ src, size_t slot_vec,
                                           uint4* __restrict__ out, size_t nvec) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i0 < nvec; i0 += stride * ROWS) {
    uint4 v[ROWS][W];
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
#pragma unroll
      for (int s = 0; s < W; ++s) {
        const size_t i = i0 + r * stride;
        v[r][s] = i < nvec ? __ldcs(src + s * slot_vec + i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int s = 0; s < W; ++s) {
        const uint32_t w[4] = {v[r][s].x, v[r][s].y, v[r][s].z, v[r][s].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[e]));
          acc[2 * e] += f.x;
          acc[2 * e + 1] += f.y;
        }
      }
      uint4 o;
      uint32_t* po = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        __nv_bfloat162 h = __floats2bfloat162_rn(acc[2 * e], acc[2 * e + 1]);
        po[e] = *reinterpret_cast<uint32_t*>(&h);
      }
      const size_t i = i0 + r * stride;
      if (i < nvec) __stcs(out + i, o);
    }
  }
}

template <int W, int ROWS>
float run(const uint4* src, size_t slot_vec, uint4* out, size_t nvec, int grid) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) red<W, ROWS><<<grid, 256>>>(src, slot_vec, out, nvec);
  cudaEventRecord(a);
  const int it = 20;
  for (int i = 0; i < it; ++i) red<W, ROWS><<<grid, 256>>>(src, slot_vec, out, nvec);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / it;
}

int main() {
  const size_t slot = 16ull << 20;  // C4 at TP=8: 1024 x 8192 bf16
  const size_t pads[] = {0, 256, 4096, 65536, 1 << 20};
  const int W = 8;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (size_t pad : pads) {
    const size_t stride = slot + pad;
    uint8_t* src;
    uint8_t* out;
    cudaMalloc(&src, stride * W);
    cudaMalloc(&out, slot);
    cudaMemset(src, 0, stride * W);
    const size_t nvec = slot / 16, svec = stride / 16;
    for (int g : {sms * 4, sms * 8, sms * 16}) {
      float t1 = run<W, 1>((const uint4*)src, svec, (uint4*)out, nvec, g);
      float t2 = run<W, 2>((const uint4*)src, svec, (uint4*)out, nvec, g);
      float t4 = run<W, 4>((const uint4*)src, svec, (uint4*)out, nvec, g);
      const double bytes = (double)slot * (W + 1);
      printf("pad=%7zu grid=%5d  rows/thread 1: %6.1f us %5.0f GB/s | 2: %6.1f us %5.0f GB/s | 4: %6.1f us %5.0f GB/s\n",
             pad, g, t1, bytes / t1 / 1e3, t2, bytes / t2 / 1e3, t4, bytes / t4 / 1e3);
    }
    cudaFree(src);
    cudaFree(out);
  }
  return 0;
}

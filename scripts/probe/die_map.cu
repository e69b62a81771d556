// Which die is each SM on?  Every SM pointer-chases (L2 hits, ld.cg) inside
// P 2-KB chunks of one buffer and records the mean latency per chunk; chunks
// homed on the SM's own die answer faster (near vs far L2).  SMs whose
// latency vectors correlate belong to the same die.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

constexpr int P = 128;        // probed 2 KB chunks
constexpr int CHASE = 64;     // dependent loads per chunk per pass
constexpr int PASSES = 4;

__global__ void probe(const unsigned* buf, float* lat, int* smid_out) {
  if (threadIdx.x != 0) return;
  unsigned sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  smid_out[blockIdx.x] = (int)sm;
  for (int c = 0; c < P; ++c) {
    const unsigned* base = buf + (size_t)c * 512 * 8;  // chunks 16 KB apart (2 KB grain)
    unsigned idx = 0;
    // warm
    for (int i = 0; i < CHASE; ++i) {
      unsigned v;
      asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(base + idx) : "memory");
      idx = v;
    }
    long long best = 1ll << 60;
    for (int pass = 0; pass < PASSES; ++pass) {
      long long t0;
      asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0) :: "memory");
      for (int i = 0; i < CHASE; ++i) {
        unsigned v;
        asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(base + idx) : "memory");
        idx = v;
      }
      long long t1;
      // the clock read consumes idx: it issues only once the last load returned
      asm volatile("add.u32 %1, %1, 0;\n\tmov.u64 %0, %%clock64;" : "=l"(t1), "+r"(idx) :: "memory");
      long long t = t1 - t0 + (idx == 0xFFFFFFFF);
      if (t < best) best = t;
    }
    lat[blockIdx.x * P + c] = (float)best / (float)CHASE + 0.001f;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t words = (size_t)P * 512 * 8;
  std::vector<unsigned> h(words, 0);
  for (int c = 0; c < P; ++c) {
    unsigned* base = h.data() + (size_t)c * 512 * 8;
    // chain through the 512 words (2 KB) of the chunk with stride 32 words (128 B lines)
    for (int i = 0; i < 16; ++i) base[i * 32] = ((i + 1) % 16) * 32;
  }
  unsigned* d; float* lat; int* smid;
  cudaMalloc(&d, words * 4); cudaMalloc(&lat, sizeof(float) * sms * P); cudaMalloc(&smid, 4 * sms);
  cudaMemcpy(d, h.data(), words * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaError_t e0 = cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  probe<<<sms, 32, 200 * 1024>>>(d, lat, smid);  // 1 block per SM (smem-limited)
  cudaError_t e1 = cudaGetLastError();
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("attr %s launch %s sync %s\n", cudaGetErrorString(e0), cudaGetErrorString(e1), cudaGetErrorString(e2));
  std::vector<float> L(sms * P); std::vector<int> S(sms);
  cudaMemcpy(L.data(), lat, sizeof(float) * sms * P, cudaMemcpyDeviceToHost);
  cudaMemcpy(S.data(), smid, 4 * sms, cudaMemcpyDeviceToHost);
  // correlate every SM's centred vector with block 0's
  auto centred = [&](int b) {
    std::vector<double> v(P); double m = 0;
    for (int c = 0; c < P; ++c) m += L[b * P + c];
    m /= P;
    for (int c = 0; c < P; ++c) v[c] = L[b * P + c] - m;
    return v;
  };
  auto r0 = centred(0);
  int same = 0;
  std::vector<int> die(sms);
  double minabs = 1;
  for (int b = 0; b < sms; ++b) {
    auto v = centred(b);
    double num = 0, a = 0, bb = 0;
    for (int c = 0; c < P; ++c) { num += v[c] * r0[c]; a += v[c] * v[c]; bb += r0[c] * r0[c]; }
    double corr = num / sqrt(a * bb + 1e-12);
    die[b] = corr > 0 ? 0 : 1;
    same += die[b] == 0;
    if (fabs(corr) < minabs) minabs = fabs(corr);
    if (b < 8 || b % 20 == 0) printf("block %3d smid %3d corr %+.3f lat[0..5] %.2f %.2f %.2f %.2f %.2f %.2f\n", b, S[b], corr,
                                     L[b*P], L[b*P+1], L[b*P+2], L[b*P+3], L[b*P+4], L[b*P+5]);
  }
  printf("die sizes: %d / %d   min |corr| %.3f\n", same, sms - same, minabs);
  printf("die by smid: ");
  std::vector<int> bysm(sms, -1);
  for (int b = 0; b < sms; ++b) if (S[b] >= 0 && S[b] < sms) bysm[S[b]] = die[b];
  for (int s = 0; s < sms; ++s) printf("%d", bysm[s]);
  printf("\n");
}

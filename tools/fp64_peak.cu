// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs DFMA.
// Not part of the product: it measures the roofline denominator the bench reports against
// (MEASURED_PEAKS.json has no fp64 entry). Build: see tools/run_peaks.sh.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;  // keep live
}

// FM x FN outer-product tile with distinct A/B fragment registers (like the GEMM main loop),
// operands perturbed every iteration so they stay live
template <int FM, int FN>
__global__ void dmma_tile_loop(double* out, int iters, double seed) {
  double a[FM], b[FN];
  double c[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i) a[i] = seed + i + threadIdx.x * 1e-3;
#pragma unroll
  for (int j = 0; j < FN; ++j) b[j] = seed - j;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][j][0]), "+d"(c[i][j][1]) : "d"(a[i]), "d"(b[j]));
    a[it % FM] = a[(it + 1) % FM];  // keep operands live without extra FP64 work
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) s += c[i][j][0] + c[i][j][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// The update-tile K loop in isolation: fragments from SMEM (conflict-free layout, ld = 4 mod 16),
// one k-step of prefetch, FM x FN accumulators; `iters` passes over a 96-deep K.
template <int FM, int FN>
__global__ void dmma_smem_loop(double* out, int iters, double seed) {
  extern __shared__ double sm[];
  constexpr int LD = 100;
  for (int i = threadIdx.x; i < 2 * 64 * LD; i += blockDim.x) sm[i] = seed + (i % 97) * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* A = sm + ((warp & 1) * 8 * FM + (lane >> 2)) * LD + (lane & 3);
  const double* B = sm + 64 * LD + ((warp >> 1) % 2 * 8 * FN + (lane >> 2)) * LD + (lane & 3);
  double acc[FN][FM][2];
#pragma unroll
  for (int j = 0; j < FN; ++j)
#pragma unroll
    for (int i = 0; i < FM; ++i) acc[j][i][0] = acc[j][i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
    double fa[2][FM], fb[2][FN];
#pragma unroll
    for (int i = 0; i < FM; ++i) fa[0][i] = A[i * 8 * LD];
#pragma unroll
    for (int j = 0; j < FN; ++j) fb[0][j] = B[j * 8 * LD];
    for (int kk = 0; kk < 96; kk += 8) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kn = kk + 4 * (h + 1);
        if (kn < 96) {
#pragma unroll
          for (int i = 0; i < FM; ++i) fa[h ^ 1][i] = A[i * 8 * LD + kn];
#pragma unroll
          for (int j = 0; j < FN; ++j) fb[h ^ 1][j] = B[j * 8 * LD + kn];
        }
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
          for (int i = 0; i < FM; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[j][i][0]), "+d"(acc[j][i][1]) : "d"(fb[h][j]), "d"(fa[h][i]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < FN; ++j)
#pragma unroll
    for (int i = 0; i < FM; ++i) s += acc[j][i][0] + acc[j][i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = 1.0 - 1e-9 * threadIdx.x;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename K>
static double time_kernel(K kern, int grid, int block, int iters, double* out, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  kern<<<grid, block>>>(out, iters, 0.5);  // warm
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<grid, block>>>(out, iters, 0.5);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

template <typename K>
static double sustained(K kern, int grid, int block, int iters, double* out, double seconds, double flop_per_launch) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  int launches = 0; float ms = 0;
  while (true) {
    for (int i = 0; i < 20; ++i) kern<<<grid, block>>>(out, iters, 0.5);
    launches += 20;
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms > seconds * 1e3) break;
  }
  return flop_per_launch * launches / (ms * 1e-3) / 1e12;
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 4096 * sizeof(double)));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"smem_optin\": %zu, \"l2\": %d", p.name, sms,
         (size_t)p.sharedMemPerBlockOptin, p.l2CacheSize);
  const int iters = 4096;
  // DMMA: per warp-instruction 8*8*4 FMA = 256 FMA = 512 flop
  int warps_list[] = {4, 8, 16};
  double best_dmma = 0;
  for (int w : warps_list) {
    int block = 32 * w, grid = sms * 2;
    double ms = time_kernel(dmma_loop<8>, grid, block, iters, out, 5);
    double flop = (double)grid * w * iters * 8 * 512.0;
    double tf = flop / (ms * 1e-3) / 1e12;
    printf(", \"dmma_w%d_tflops\": %.3f", w, tf);
    if (tf > best_dmma) best_dmma = tf;
  }
  {
    int ws[] = {4, 8, 12, 16};
    for (int w : ws) {
      int block = 32 * w, grid = sms;
      double ms = time_kernel(dmma_tile_loop<3, 6>, grid, block, 1024, out, 5);
      double flop = (double)grid * w * 1024 * 18 * 512.0;
      printf(", \"dmma_tile3x6_w%d_tflops\": %.3f", w, flop / (ms * 1e-3) / 1e12);
      ms = time_kernel(dmma_tile_loop<6, 4>, grid, block, 1024, out, 5);
      flop = (double)grid * w * 1024 * 24 * 512.0;
      printf(", \"dmma_tile6x4_w%d_tflops\": %.3f", w, flop / (ms * 1e-3) / 1e12);
      ms = time_kernel(dmma_tile_loop<3, 3>, grid, block, 1024, out, 5);
      flop = (double)grid * w * 1024 * 9 * 512.0;
      printf(", \"dmma_tile3x3_w%d_tflops\": %.3f", w, flop / (ms * 1e-3) / 1e12);
      ms = time_kernel(dmma_tile_loop<4, 4>, grid, block, 1024, out, 5);
      flop = (double)grid * w * 1024 * 16 * 512.0;
      printf(", \"dmma_tile4x4_w%d_tflops\": %.3f", w, flop / (ms * 1e-3) / 1e12);
    }
  }
  {
    int ws[] = {4, 8, 12, 16};
    for (int w : ws) {
      int block = 32 * w, grid = sms;
      size_t smem = 2 * 64 * 100 * 8;
      cudaFuncSetAttribute(dmma_smem_loop<6, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(dmma_smem_loop<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      dmma_smem_loop<6, 3><<<grid, block, smem>>>(out, 200, 0.5);
      cudaEventRecord(e0); dmma_smem_loop<6, 3><<<grid, block, smem>>>(out, 200, 0.5); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = (double)grid * w * 200 * 24 * 18 * 512.0;
      printf(", \"dmma_smem6x3_w%d_tflops\": %.3f", w, flop / (ms * 1e-3) / 1e12);
      dmma_smem_loop<4, 4><<<grid, block, smem>>>(out, 200, 0.5);
      cudaEventRecord(e0); dmma_smem_loop<4, 4><<<grid, block, smem>>>(out, 200, 0.5); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      flop = (double)grid * w * 200 * 24 * 16 * 512.0;
      printf(", \"dmma_smem4x4_w%d_tflops\": %.3f", w, flop / (ms * 1e-3) / 1e12);
    }
  }
  double best_dfma = 0;
  for (int w : warps_list) {
    int block = 32 * w, grid = sms * 2;
    double ms = time_kernel(dfma_loop<16>, grid, block, iters, out, 5);
    double flop = (double)grid * block * iters * 16 * 2.0;
    double tf = flop / (ms * 1e-3) / 1e12;
    printf(", \"dfma_w%d_tflops\": %.3f", w, tf);
    if (tf > best_dfma) best_dfma = tf;
  }
  {
    int w = 8, block = 256, grid = sms * 2;
    double flop = (double)grid * w * iters * 8 * 512.0;
    printf(", \"dmma_sustained_tflops\": %.3f", sustained(dmma_loop<8>, grid, block, iters, out, 4.0, flop));
    double flop2 = (double)grid * block * iters * 16 * 2.0;
    printf(", \"dfma_sustained_tflops\": %.3f", sustained(dfma_loop<16>, grid, block, iters, out, 4.0, flop2));
  }
  printf(", \"dmma_burst_tflops\": %.3f, \"dfma_burst_tflops\": %.3f}\n", best_dmma, best_dfma);
  return 0;
}

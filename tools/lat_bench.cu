// Latency microbenchmark (one warp): dependent DFMA / DADD chains, MUFU.RSQ64H, SMEM load->store
// round trips.  Informs the chase design (a chain of small dependent reflectors).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_bench tools/lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double* out, long long* cyc, double a, double b, int iters) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, b, a);  // dependent DFMA
  long long t1 = clock64();
  double y = x;
  for (int i = 0; i < iters; ++i) {
    double r;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
    y = r + 1.0;
  }
  long long t2 = clock64();
  // smem: dependent load -> fma -> store -> load of the same word
  const int idx = threadIdx.x * 3;
  double z = 0.0;
  for (int i = 0; i < iters; ++i) {
    volatile double* vs = s;
    z = vs[idx];
    vs[idx] = fma(z, b, a);
  }
  long long t3 = clock64();
  // 3 loads, 4-op chain, 3 stores (one left-apply column), repeated on the same column
  double* c = s + (threadIdx.x & 15) * 33;
  const double v1 = 0.3, v2 = 0.2, tau = 1.1;
  for (int i = 0; i < iters; ++i) {
    const double h0 = c[0], h1 = c[1], h2 = c[2];
    const double tw = tau * fma(v2, h2, fma(v1, h1, h0));
    c[0] = h0 - tw;
    c[1] = fma(-tw, v1, h1);
    c[2] = fma(-tw, v2, h2);
    __syncwarp();
  }
  long long t4 = clock64();
  out[threadIdx.x] = x + y + z + c[0];
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 8 * sizeof(long long));
  const int iters = 4096;
  for (int r = 0; r < 2; ++r) lat<<<1, 32>>>(out, cyc, 1e-3, 0.999, iters);
  cudaDeviceSynchronize();
  printf("per op (cycles): DFMA %.1f  RSQ64H+DADD %.1f  LDS->DFMA->STS %.1f  left-apply column %.1f\n",
         (double)cyc[0] / iters, (double)cyc[1] / iters, (double)cyc[2] / iters, (double)cyc[3] / iters);
  return 0;
}

// Latency microbenchmark of the chase's reflector computation (one warp, dependent chain):
// cycles per house() for the product variant and alternatives.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include "../paper_2007_03576_b200/csrc/device_common.cuh"

using namespace hqr;

__device__ __forceinline__ double rsqrt_f32seed(double s) {
  double y = (double)rsqrtf((float)s);
  const double hs = 0.5 * s;
  y = y * fma(-hs * y, y, 1.5);
  y = y * fma(-hs * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double rcp_f32seed(double q) {
  double r = (double)__frcp_rn((float)q);
  r = r * fma(-q, r, 2.0);
  r = r * fma(-q, r, 2.0);
  return fma(r, fma(-q, r, 1.0), r);
}

// one Newton step fewer each: rsqrt 1 step (the sqrt correction squares its error again), rcp 1 step
// + the final correction
__device__ __forceinline__ double rsqrt_nr1(double s) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s));
  return y * fma(-0.5 * s * y, y, 1.5);
}
__device__ __forceinline__ double rcp_nr1(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  r = r * fma(-q, r, 2.0);
  return fma(r, fma(-q, r, 1.0), r);
}

template <int V>
__device__ __forceinline__ void house_v(double x0, double x1, double x2, double& v1, double& v2, double& tau,
                                        double& beta) {
  if (V == 0) { house(x0, x1, x2, v1, v2, tau, beta); return; }
  const double amax = fmax(fabs(x0), fmax(fabs(x1), fabs(x2)));
  const long long E = __double_as_longlong(amax) >> 52;
  const bool ok = (E >= 1) & (E <= 2044);
  const double down = ok ? __longlong_as_double((2045 - E) << 52) : 1.0;
  x1 *= down; x2 *= down;
  const double tail2 = fma(x1, x1, x2 * x2);
  if (tail2 == 0.0) { v1 = 0.0; v2 = 0.0; tau = 0.0; beta = x0; return; }
  const double xs0 = x0 * down;
  const double s = fma(xs0, xs0, tail2);
  double nrm, r;
  if (V == 1 || V == 3) {
    const double y = V == 1 ? rsqrt_f32seed(s) : rsqrt_nr1(s);
    nrm = s * y;
    nrm = fma(0.5 * y, fma(-nrm, nrm, s), nrm);
  } else {
    nrm = sqrt(s);
  }
  const double b = (xs0 >= 0.0) ? -nrm : nrm;
  const double d = xs0 - b;
  if (V == 1) r = rcp_f32seed(d * b); else if (V == 3) r = rcp_nr1(d * b); else r = 1.0 / (d * b);
  const double br = b * r;
  v1 = x1 * br; v2 = x2 * br; tau = -d * d * r;
  beta = b * (ok ? __longlong_as_double((E + 1) << 52) : 1.0);
}

// burst mode (the chase's phase 1): every warp computes one reflector per barrier interval; LANE1:
// only lane 0 computes, the results are broadcast with shuffles
template <bool LANE1>
__global__ void burst(double* out, long long* cyc, int iters) {
  __shared__ double xs[16][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane < 3) xs[warp][lane] = 1.0 + lane * 0.5 + warp * 1e-3;
  __syncthreads();
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double x0 = xs[warp][0], x1 = xs[warp][1], x2 = xs[warp][2];
    double v1 = 0, v2 = 0, tau = 0, beta = 0;
    if (!LANE1 || lane == 0) house(x0, x1, x2, v1, v2, tau, beta);
    if (LANE1) {
      v1 = __shfl_sync(0xffffffffu, v1, 0); v2 = __shfl_sync(0xffffffffu, v2, 0);
      tau = __shfl_sync(0xffffffffu, tau, 0); beta = __shfl_sync(0xffffffffu, beta, 0);
    }
    acc += v1 + v2 + tau;
    __syncwarp();
    if (lane == 0) { xs[warp][0] = beta * -0.7 + 1.5; xs[warp][1] = v2 + 0.3; xs[warp][2] = tau * 0.2 + 0.1; }
    __syncthreads();
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / iters;
}

template <int V>
__global__ void k(double* out, long long* cyc, int iters) {
  double x0 = 1.0 + threadIdx.x * 1e-3, x1 = 0.5, x2 = 0.25;
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double v1, v2, tau, beta;
    house_v<V>(x0, x1, x2, v1, v2, tau, beta);
    x0 = beta * -0.7 + v1; x1 = v2 + 0.3; x2 = tau * 0.2 + 0.1;  // dependent chain
    acc += tau;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc + x0 + x1 + x2;
  if (threadIdx.x == 0) *cyc = (t1 - t0) / iters;
}

// accuracy against the IEEE variant (V = 2) on inputs over a wide exponent range: max |diff| / |ref|
// in units of 2^-53 for v1, v2, tau, beta
template <int V>
__global__ void acc_k(unsigned long long* worst, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long x = 0x9E3779B97F4A7C15ull * (i + 1);
  auto rnd = [&]() { x ^= x >> 12; x ^= x << 25; x ^= x >> 27; return (double)((x * 2685821657736338717ull) >> 11) * 0x1.0p-53; };
  const int e = (int)(rnd() * 400) - 200;
  const double sc = ldexp(1.0, e);
  const double x0 = (rnd() - 0.5) * sc, x1 = (rnd() - 0.5) * sc * ldexp(1.0, (int)(rnd() * 40) - 20), x2 = (rnd() - 0.5) * sc;
  double a[4], b[4];
  house_v<V>(x0, x1, x2, a[0], a[1], a[2], a[3]);
  house_v<2>(x0, x1, x2, b[0], b[1], b[2], b[3]);
  for (int k = 0; k < 4; ++k) {
    const double r = b[k] == 0.0 ? 0.0 : fabs(a[k] - b[k]) / fabs(b[k]) * 0x1.0p53;
    atomicMax(&worst[k], (unsigned long long)(r * 1000.0));
  }
}

int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
  const char* names[3] = {"product house (rsqrt/rcp.approx.f64 + Newton)", "float-seeded rsqrtf/frcp + f64 Newton", "IEEE sqrt + division"};
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 32>>>(out, cyc, 1000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); if (rep) printf("%-50s %lld cycles/house\n", names[0], h);
    k<1><<<1, 32>>>(out, cyc, 1000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); if (rep) printf("%-50s %lld cycles/house\n", names[1], h);
    k<2><<<1, 32>>>(out, cyc, 1000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); if (rep) printf("%-50s %lld cycles/house\n", names[2], h);
  }
  // 13 warps concurrently (the fused chase): per-warp cycles
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 416>>>(out, cyc, 1000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); if (rep) printf("13 warps: %-40s %lld\n", names[0], h);
    k<1><<<1, 416>>>(out, cyc, 1000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); if (rep) printf("13 warps: %-40s %lld\n", names[1], h);
  }
  for (int rep = 0; rep < 2; ++rep) {
    burst<false><<<1, 416>>>(out, cyc, 1000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); if (rep) printf("burst 13 warps, all lanes:  %lld cycles per reflector + barrier\n", h);
    burst<true><<<1, 416>>>(out, cyc, 1000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); if (rep) printf("burst 13 warps, lane 0 + shfl: %lld\n", h);
    burst<false><<<1, 32>>>(out, cyc, 1000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); if (rep) printf("burst 1 warp, all lanes:  %lld\n", h);
  }
  {
    unsigned long long* w; unsigned long long hw[4];
    cudaMalloc(&w, 32);
    const char* vn[2] = {"product", "one Newton step fewer"};
    for (int v = 0; v < 2; ++v) {
      cudaMemset(w, 0, 32);
      if (v == 0) acc_k<0><<<4096, 256>>>(w, 1 << 20); else acc_k<3><<<4096, 256>>>(w, 1 << 20);
      cudaMemcpy(hw, w, 32, cudaMemcpyDeviceToHost);
      printf("accuracy %-24s max rel diff vs IEEE (units of 2^-53): v1 %.3f v2 %.3f tau %.3f beta %.3f\n", vn[v],
             hw[0] / 1000.0, hw[1] / 1000.0, hw[2] / 1000.0, hw[3] / 1000.0);
    }
    for (int rep = 0; rep < 2; ++rep) {
      k<3><<<1, 32>>>(out, cyc, 1000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); if (rep) printf("%-50s %lld cycles/house\n", "one Newton step fewer", h);
      k<3><<<1, 416>>>(out, cyc, 1000); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); if (rep) printf("13 warps: %-40s %lld\n", "one Newton step fewer", h);
    }
  }
  return 0;
}

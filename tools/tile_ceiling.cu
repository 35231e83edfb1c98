// tools/tile_ceiling.cu -- in-tile DMMA ceiling of the product update tile (gemm_tile.cuh
// consume_tile): one CTA per SM, three consumer groups of four warps (the fused kernel's layout),
// each group multiplying its SMEM-resident panel tile by the SMEM-resident band-trimmed Q_W over and
// over (no producer, no TMA, no dependencies, no chase).  Executed DMMA TFLOP/s = the ceiling the
// fused kernel's tile code allows; the gap between it and the fused kernel's 28 TF/s is scheduling.
// Not part of the product.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr [-DHQR_BENCH_NO_STORE]
//        -o tools/tile_ceiling tools/tile_ceiling.cu -lcuda
#include <cstdio>
#include <vector>
#include <algorithm>

#include "../paper_2007_03576_b200/csrc/gemm_tile.cuh"

using namespace hqr;
constexpr int KP = 96;
constexpr int QLD = pad_ld(KP);
constexpr int SS = Geom<KP, true>::STAGE > Geom<KP, false>::STAGE ? Geom<KP, true>::STAGE : Geom<KP, false>::STAGE;

template <bool LEFT>
__global__ void __launch_bounds__(416) ceil_k(const double* qsrc, const double* psrc, double* out, int reps,
                                              int rotate) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ uint64_t empty[3];
  double* Qs = reinterpret_cast<double*>(smraw);
  double* Ps = Qs + KP * QLD;
  for (int i = threadIdx.x; i < KP * QLD; i += blockDim.x) Qs[i] = qsrc[i];
  for (int i = threadIdx.x; i < 3 * SS; i += blockDim.x) Ps[i] = psrc[i % SS];
  if (threadIdx.x < 3) mbar_init(&empty[threadIdx.x], 4);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= 12) return;
  const int q = warp >> 2, i4 = warp & 3;
  TileRef t;
  t.w0 = 0; t.kw = KP; t.nbc = 13;
  t.M = out + (size_t)blockIdx.x * 3 * 3072 + q * 3072;
  t.c0 = 0; t.lc1 = 32; t.ld = LEFT ? KP : 32; t.cb = 0; t.r0 = 0; t.r1 = 32; t.isZ = false;
  for (int r = 0; r < reps; ++r) {
    const int qq = rotate ? (i4 + r + q) & 3 : i4;
    consume_tile<KP, LEFT>(Qs, Ps + q * SS, &empty[q], t, qq, lane);
    if (rotate == 2) named_sync(1 + q, 128);  // a group's warps in lock step (the ring's coupling, tight)
  }
}

int main(int argc, char** argv) {
  const int nbc = argc > 1 ? atoi(argv[1]) : 13;
  const int reps = argc > 2 ? atoi(argv[2]) : 2000;
  const int kw = KP, sw = kw - 3 * nbc - 1;
  // Q_W band as the chase leaves it (tools/gemm_bench.cu): rows c - s - 1 .. c + 2 nbc of column c
  std::vector<double> hq((size_t)KP * QLD, 0.0), hp(SS);
  double units = 0;  // executed (8-column block x K row) units
  for (int c = 0; c < kw; ++c)
    for (int k = 0; k < kw; ++k)
      if (k <= c + 2 * nbc && k >= c - sw - 1) hq[k + (size_t)c * QLD] = ((k * 7 + c * 13) % 17 + 1) / 17.0 - 0.5;
  for (int b = 0; b < KP / 8; ++b) {
    int lo = 1 << 30, hi = -1;
    for (int c = 8 * b; c < 8 * b + 8; ++c)
      for (int k = 0; k < KP; ++k)
        if (hq[k + (size_t)c * QLD] != 0.0) { lo = std::min(lo, k); hi = std::max(hi, k); }
    const double klo = hi < 0 ? 0 : (lo & ~3), khi = hi < 0 ? 0 : ((hi + 4) & ~3);
    hq[KP + (size_t)8 * b * QLD] = klo;
    hq[KP + 1 + (size_t)8 * b * QLD] = khi;
    units += khi - klo;
  }
  for (int i = 0; i < SS; ++i) hp[i] = ((i * 31) % 29) / 29.0 - 0.5;
  double *dq, *dp, *dout;
  cudaMalloc(&dq, hq.size() * 8);
  cudaMalloc(&dp, SS * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&dout, (size_t)sms * 3 * 3072 * 8);
  cudaMemcpy(dq, hq.data(), hq.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, hp.data(), SS * 8, cudaMemcpyHostToDevice);
  const size_t smem = (size_t)(KP * QLD + 3 * SS) * 8;
  cudaFuncSetAttribute(ceil_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(ceil_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 6; ++mode) {
    const bool left = mode % 2 == 0;
    const int rot = mode / 2 == 0 ? 0 : mode / 2 == 1 ? 1 : 2;
    auto launch = [&]() {
      if (left) ceil_k<true><<<sms, 416, smem>>>(dq, dp, dout, reps, rot);
      else ceil_k<false><<<sms, 416, smem>>>(dq, dp, dout, reps, rot);
    };
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    // executed flops per tile: every 8-column block b over its K extent x the tile's other side (32)
    const double tile_fl = units * 8.0 * 32.0 * 2.0;
    const double fl = (double)sms * 3 * reps * tile_fl;
    printf("{\"tile\": \"%s\", \"quarters\": \"%s\", \"nbc\": %d, \"exec_frac\": %.3f, \"ms\": %.3f, "
           "\"exec_tflops\": %.2f, \"err\": \"%s\"}\n", left ? "left" : "right", rot == 0 ? "fixed" : rot == 1 ? "rotating" : "rotating, group lock step",
           nbc, units * 8.0 / (KP * KP), ms, fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

// tools/gemm_bench.cu -- isolated timing of the update kernels (update.cu) on a synthetic step.
// Not part of the product.  Build: see tools/run_gemm_bench.sh.  Prints JSON lines.
//   n, C windows of side kw at the given spacing, random Q_W (lower bandwidth 2*nbc), random H/Z.
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#include "../paper_2007_03576_b200/csrc/update.cu"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void fill(double* p, size_t n, unsigned seed) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (x & 0xffffff) / 16777216.0 - 0.5;
  }
}

int main(int argc, char** argv) {
  int64_t n = argc > 1 ? atoll(argv[1]) : 20000;
  int C = argc > 2 ? atoi(argv[2]) : 18;
  int kw = argc > 3 ? atoi(argv[3]) : 96;
  int nbc = argc > 4 ? atoi(argv[4]) : 15;
  int64_t pos = argc > 5 ? atoll(argv[5]) : 8000;  // w0 of the top window
  int reps = argc > 6 ? atoi(argv[6]) : 20;
  int KP = hqr::padded_kp(kw), QLD = hqr::pad_ld(KP);
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  double *H, *Z, *Q;
  CK(cudaMalloc(&H, n * n * 8));
  CK(cudaMalloc(&Z, n * n * 8));
  CK(cudaMalloc(&Q, (size_t)C * KP * QLD * 8));
  fill<<<1024, 256>>>(H, n * n, 1);
  fill<<<1024, 256>>>(Z, n * n, 2);
  // Q slots: random inside the band of a real window (rows c - s - 1 .. c + 2 nbc of column c,
  // s = kw - 3 nbc - 1), zero elsewhere; per-8-column-block K extents in the padding rows (as
  // store_q_slot writes them).  exec_frac = executed / dense DMMA work.
  std::vector<double> hq((size_t)C * KP * QLD, 0.0);
  const int sw = kw - 3 * nbc - 1;
  double exec_frac = 0.0;
  for (int s = 0; s < C; ++s) {
    double* qs = hq.data() + (size_t)s * KP * QLD;
    for (int c = 0; c < kw; ++c)
      for (int k = 0; k < kw; ++k)
        if (k <= c + 2 * nbc && k >= c - sw - 1) qs[k + (size_t)c * QLD] = ((k * 7 + c * 13 + s) % 17 + 1) / 17.0 - 0.5;
    for (int b = 0; b < KP / 8; ++b) {
      int lo = 1 << 30, hi = -1;
      for (int c = 8 * b; c < 8 * b + 8; ++c)
        for (int k = 0; k < KP; ++k)
          if (qs[k + (size_t)c * QLD] != 0.0) { lo = std::min(lo, k); hi = std::max(hi, k); }
      double klo = hi < 0 ? 0 : (lo & ~3), khi = hi < 0 ? 0 : ((hi + 4) & ~3);
      qs[KP + (size_t)8 * b * QLD] = klo;
      qs[KP + 1 + (size_t)8 * b * QLD] = khi;
      if (s == 0) exec_frac += 8.0 * (khi - klo) / ((double)KP * KP);
    }
  }
  CK(cudaMemcpy(Q, hq.data(), hq.size() * 8, cudaMemcpyHostToDevice));
  std::vector<hqr::WindowDesc> w(C);
  int lag_s = (kw + 4);
  for (int c = 0; c < C; ++c) {
    w[c].chain = C - 1 - c;
    w[c].w0 = (int)(pos + (int64_t)c * lag_s);
    w[c].w1 = w[c].w0 + kw - 1;
    w[c].t0 = 0; w[c].t1 = 0; w[c].b0 = 0; w[c].nbc = nbc; w[c].slot = c; w[c].last = 0;
  }
  hqr::WindowDesc* dw;
  CK(cudaMalloc(&dw, C * sizeof(hqr::WindowDesc)));
  CK(cudaMemcpy(dw, w.data(), C * sizeof(hqr::WindowDesc), cudaMemcpyHostToDevice));
  hqr::StepArgs a{};
  a.H = H; a.Z = Z; a.n = n; a.ilo = 0; a.ihi = n - 1; a.wins = dw; a.win_begin = 0; a.win_count = C;
  a.qslots = Q; a.KP = KP; a.QLD = QLD; a.slot_offset = 0;
  a.hcol0 = 0; a.lc0 = 0; a.lc1 = n; a.zrows = n; a.ldz = n;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  hqr::TensorMaps tm;
  CK(hqr::make_tensor_maps(&tm, H, n, Z, n, n, n, KP));
  {
    const unsigned long long* q = reinterpret_cast<const unsigned long long*>(&tm.left_H);
    fprintf(stderr, "bench: tensor maps valid=%d KP=%d H=%p map@%p %llx %llx %llx\n", (int)tm.valid, KP,
            (const void*)H, (const void*)&tm.left_H, q[0], q[1], q[2]);
  }
  const char* names[3] = {"left", "right_H", "right_Z"};
  for (int mode = 0; mode < 3; ++mode) {
    int64_t items; double fl, by;
    hqr::StepArgs b = a;
    b.right_mode = mode == 1 ? 1 : 2;
    auto launch = [&]() {
      if (mode == 0) CK(hqr::launch_left(b, w.data(), prop.multiProcessorCount, tm, 0, &items, &fl, &by));
      else CK(hqr::launch_right(b, w.data(), prop.multiProcessorCount, tm, 0, &items, &fl, &by));
    };
    launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    // executed DMMA flops (K trimmed per warp as in the kernel) ~ dense * trim; report dense
    printf("{\"kernel\": \"%s\", \"n\": %lld, \"C\": %d, \"kw\": %d, \"nbc\": %d, \"items\": %lld, \"ms\": %.4f, "
           "\"dense_tflops\": %.3f, \"exec_frac\": %.3f, \"hbm_gbs\": %.1f}\n",
           names[mode], (long long)n, C, kw, nbc, (long long)items, ms, fl / (ms * 1e-3) / 1e12, exec_frac,
           by / (ms * 1e-3) / 1e9);
  }
  return 0;
}

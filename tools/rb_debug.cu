// Diagnostic: k_rebuild (tensor-core V rebuild) against the streaming
// k_extend<8> passes on a synthetic factor, element by element.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I include -o tools/rb_debug tools/rb_debug.cu
#include "../paper_2111_14991_b200/csrc/gtc_kernels.cu"

#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

int main(int argc, char** argv) {
  using namespace gtc;
  const int n = argc > 1 ? std::atoi(argv[1]) : 64;
  const int d = 3;
  const int64_t N = 4096, n_pad = 4096;
  std::mt19937_64 g(11);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<double> coords(d * n_pad), tx(n * d), tn2(n), L(packed(n) + 8, 0.0);
  for (auto& x : coords) x = U(g);
  for (auto& x : tx) x = U(g);
  for (int i = 0; i < n; ++i) {
    double s = 0;
    for (int t = 0; t < d; ++t) s = s + tx[i * d + t] * tx[i * d + t];
    tn2[i] = s;
    for (int j = 0; j < i; ++j) L[packed(i) + j] = 0.3 * (U(g) - 0.5);
    L[packed(i) + i] = 0.5 + U(g);
  }
  double *dc, *dtx, *dtn2, *dL, *V1, *V2;
  const int64_t tile_stride = (int64_t)n * kTile;
  cudaMalloc(&dc, 8 * coords.size()); cudaMalloc(&dtx, 8 * tx.size()); cudaMalloc(&dtn2, 8 * n);
  cudaMalloc(&dL, 8 * L.size()); cudaMalloc(&V1, 8 * tile_stride * (n_pad / kTile)); cudaMalloc(&V2, 8 * tile_stride * (n_pad / kTile));
  cudaMemcpy(dc, coords.data(), 8 * coords.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dtx, tx.data(), 8 * tx.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dtn2, tn2.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dL, L.data(), 8 * L.size(), cudaMemcpyHostToDevice);
  SpaceDev sp{dc, N, n_pad, d, nullptr, nullptr};
  GpDev gd{};
  gd.train_x = dtx; gd.train_n2 = dtn2; gd.L = dL; gd.n_max = n; gd.d = d;
  KernelParams kp{1, 0.7, 1.3};
  for (int n0 = 0; n0 < n; n0 += kMaxRows)
    launch_extend(sp, gd, kp, V1, tile_stride, n0, std::min(kMaxRows, n - n0), false, nullptr, nullptr, false, nullptr, nullptr, 0);
  set_rebuild_mode(1);
  const bool ok = launch_rebuild(sp, gd, kp, V2, tile_stride, n, 0);
  cudaDeviceSynchronize();
  std::printf("rebuild taken %d err %s\n", ok, cudaGetErrorString(cudaGetLastError()));
  std::vector<double> h1(tile_stride * (n_pad / kTile)), h2(h1.size());
  cudaMemcpy(h1.data(), V1, 8 * h1.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), V2, 8 * h2.size(), cudaMemcpyDeviceToHost);
  long bad = 0;
  int shown = 0;
  std::vector<long> row_bad(n, 0);
  for (int64_t t = 0; t < n_pad / kTile; ++t)
    for (int r = 0; r < n; ++r)
      for (int c = 0; c < kTile; ++c) {
        const int64_t i = t * tile_stride + (int64_t)r * kTile + c;
        if (std::memcmp(&h1[i], &h2[i], 8)) {
          ++bad;
          ++row_bad[r];
          if (shown++ < 5) std::printf("tile %ld row %d cand %d: %.17g vs %.17g\n", (long)t, r, c, h1[i], h2[i]);
        }
      }
  std::printf("n %d mismatches %ld of %ld\n", n, bad, (long)h1.size());
  for (int r = 0; r < n; ++r) if (row_bad[r]) { std::printf("first bad row %d (%ld)\n", r, row_bad[r]); break; }
  return 0;
}

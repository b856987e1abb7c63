// Diagnostic: times the selection kernel alone on a dumped run state
// (tools/dump_state.py -> /tmp/gtc_state.bin), compiled with -DGTC_SEL_STOP=k
// to cut the kernel after a phase.  Not part of the product.
#include "../paper_2111_14991_b200/csrc/gtc_kernels.cu"

#include <cstdio>
#include <algorithm>
#include <vector>

int main(int argc, char** argv) {
  const char* path = argc > 1 ? argv[1] : "/tmp/gtc_state.bin";
  FILE* f = fopen(path, "rb");
  if (!f) { printf("no state file\n"); return 1; }
  int64_t n;
  double best_raw, ymean, ystd, mu_s, var_s;
  fread(&n, 8, 1, f);
  fread(&best_raw, 8, 1, f); fread(&ymean, 8, 1, f); fread(&ystd, 8, 1, f);
  fread(&mu_s, 8, 1, f); fread(&var_s, 8, 1, f);
  std::vector<double> mu(n), var(n);
  std::vector<uint32_t> vis((n + 31) / 32);
  fread(mu.data(), 8, n, f); fread(var.data(), 8, n, f); fread(vis.data(), 4, vis.size(), f);
  fclose(f);
  double *dmu, *dvar;
  uint32_t* dvis;
  cudaMalloc(&dmu, 8 * n); cudaMalloc(&dvar, 8 * n); cudaMalloc(&dvis, 4 * vis.size());
  cudaMemcpy(dmu, mu.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dvar, var.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dvis, vis.data(), 4 * vis.size(), cudaMemcpyHostToDevice);
  // variance total over the unvisited candidates (passed by value)
  const int np = (int)((n + 255) / 256);
  std::vector<double> hps(np, 0.0);
  std::vector<long long> hpc(np, 0);
  for (int64_t j = 0; j < n; ++j)
    if (!((vis[j >> 5] >> (j & 31)) & 1u)) { hps[j / 256] += var[j]; hpc[j / 256]++; }
  double tsum = 0.0;
  long long tcnt = 0;
  for (int t = 0; t < np; ++t) { tsum += hps[t]; tcnt += hpc[t]; }
  const gtc::VarSource vs{nullptr, 1.0, tsum, tcnt, 1};
  // tile summaries as the pass leaves them; first eligible + count as the host computes them
  std::vector<gtc::TileStats> hts(np);
  for (int t = 0; t < np; ++t) {
    double mn = 1e300, vx = -1.0, vn = 1e300, va = 0.0;
    int64_t mp = -1;
    double sm = 1e300;
    for (int64_t j = (int64_t)t * 256; j < std::min<int64_t>(n, (int64_t)(t + 1) * 256); ++j) {
      mn = std::min(mn, mu[j]);
      const bool u = !((vis[j >> 5] >> (j & 31)) & 1u);
      if (u && (mp < 0 || mu[j] < sm)) { sm = mu[j]; va = var[j]; mp = j; }
      vx = std::max(vx, var[j]); vn = std::min(vn, var[j]);
    }
    hts[t] = gtc::TileStats{mn, vx, vn, sm, va, mp};
  }
  gtc::TileStats* dts;
  cudaMalloc(&dts, sizeof(gtc::TileStats) * np);
  cudaMemcpy(dts, hts.data(), sizeof(gtc::TileStats) * np, cudaMemcpyHostToDevice);
  int64_t first = -1;
  for (int64_t j = 0; j < n && first < 0; ++j) if (!((vis[j >> 5] >> (j & 31)) & 1u)) first = j;
  gtc::GpScalars* sc;
  cudaMallocManaged(&sc, sizeof(gtc::GpScalars));
  memset(sc, 0, sizeof(*sc));
  sc->y_mean = ymean; sc->y_std = ystd;
  gtc::ReduceBufs b{};
  cudaMalloc(&b.pscore, 8 * 3 * 4096); cudaMalloc(&b.ppos, 8 * 3 * 4096);
  cudaMalloc(&b.pfirst, 8 * 4096); cudaMalloc(&b.pcnt, 8 * 4096); cudaMalloc(&b.pfinite, 4 * 4096);
  cudaMalloc(&b.counter, 4); cudaMemset(b.counter, 0, 4);
  cudaMalloc(&b.gthr, 24); cudaMemset(b.gthr, 0, 24);
  gtc::SelectDev* out;
  cudaMallocManaged(&out, sizeof(gtc::SelectDev));
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  double* flush;
  const size_t fl = 256ull << 20;
  cudaMalloc(&flush, fl);
  for (uint32_t mask : {1u, 2u, 4u, 7u}) {
    gtc::SelectParams p{mask, 1, 0.01, mu_s, var_s, best_raw, nullptr, 0, first, tcnt};
    float tot = 0.f;
    const int reps = 50;
    for (int r = 0; r < reps + 3; ++r) {
      cudaMemsetAsync(flush, r, fl, s);  // evict L2 like the V stream does
      cudaEventRecord(e0, s);
      gtc::launch_select(dmu, dvar, dvis, n, sc, p, vs, dts, b, out, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 3) tot += ms;
    }
#ifdef GTC_SEL_TRACE
    {
      unsigned long long tr[2048][8];
      cudaMemcpyFromSymbol(tr, gtc::g_sel_trace, sizeof(tr));
      const char* ge = getenv("GTC_SELECT_GRID");
      const int grid = std::min(np, ge ? atoi(ge) : (mask & (mask - 1) ? 1 : 2) * 148);
      unsigned long long t0 = ~0ull, tend = 0;
      for (int bk = 0; bk < grid; ++bk) t0 = tr[bk][0] < t0 ? tr[bk][0] : t0;
      double acc[8] = {0}, mx[8] = {0};
      for (int bk = 0; bk < grid; ++bk)
        for (int k = 0; k < 6; ++k) {
          const double v = (tr[bk][k] - t0) / 1e3;
          acc[k] += v / grid;
          mx[k] = v > mx[k] ? v : mx[k];
        }
      for (int bk = 0; bk < grid; ++bk) if (tr[bk][6] > tend) tend = tr[bk][6];
      printf("trace mask=%u grid=%d avg/max us: start %.2f/%.2f setup %.2f/%.2f seed %.2f/%.2f cands %.2f/%.2f blockdone %.2f/%.2f end %.2f\n",
             mask, grid, acc[0], mx[0], acc[1], mx[1], acc[2], mx[2], acc[3], mx[3], acc[5], mx[5], (tend - t0) / 1e3);
    }
#endif
    printf("mask=%u  %.2f us  pos=%lld,%lld,%lld lambda=%.6g err=%s\n", mask,
           1e3 * tot / reps, (long long)out->position[0], (long long)out->position[1],
           (long long)out->position[2], out->lambda, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

// Phase cycles of the one-cluster small Cholesky (small.cu, SF_SMALL_TIMING), n = 256, s = 16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSF_SMALL_TIMING -I include \
//        -I paper_1812_02056_b200/csrc calib/small_probe.cu -o calib/small_probe
#include <cstdio>
#include <vector>
#include "../paper_1812_02056_b200/csrc/small.cu"
namespace sf { void count_launch(int) {} }
int main() {
  using namespace sf;
  const int n = 256, s = 16;
  std::vector<double> h(n * n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) h[i + j * n] = (i == j) ? n : ((i * 7 + j * 13) % 17 - 8) / 17.0 + ((j * 7 + i * 13) % 17 - 8) / 17.0;
  double *d, *l; long long* fail;
  cudaMalloc(&d, n * n * 8); cudaMalloc(&l, n * n * 8); cudaMalloc(&fail, 16);
  cudaMemcpy(d, h.data(), n * n * 8, cudaMemcpyHostToDevice);
  const char* names[] = {"load", "panel", "bar1", "copy", "flush", "bar2", "store"};
  for (int rep = 0; rep < 2; ++rep) {
    long long init[2] = {kNoFail, 0};
    cudaMemcpy(fail, init, 16, cudaMemcpyHostToDevice);
    unsigned long long z[8][16][8] = {};
    cudaMemcpyToSymbol(small_times, z, sizeof(z));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = chol_small(n, s, d, n, l, n, fail, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long t[8][16][8];
    cudaMemcpyFromSymbol(t, small_times, sizeof(t));
    printf("rep %d: %.1f us (%s / %s)\n", rep, ms * 1000, cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
    for (int k = 0; k < 8; ++k) {
      printf("  cta %d:", k);
      for (int p = 0; p < 7; ++p) {
        unsigned long long mn = ~0ull, mx = 0; int wmx = 0;
        for (int w = 0; w < 8; ++w) { if (t[w][k][p] > mx) { mx = t[w][k][p]; wmx = w; } if (t[w][k][p] < mn) mn = t[w][k][p]; }
        printf(" %s %.1f-%.1f(w%d)", names[p], mn / 1965.0, mx / 1965.0, wmx);
      }
      printf(" (us)\n");
    }
  }
  {
    unsigned long long st[8][40][3];
    cudaMemcpyFromSymbol(st, small_steps, sizeof(st));
    for (int k = 0; k < 8; k += 7)
      for (int q = 0; q < 16; ++q)
        printf("cta %d step %2d: panel_end %8.2f bar1_end %8.2f step_end %8.2f (us from step 0 panel end)\n", k, q,
               ((long long)st[k][q][0] - (long long)st[k][0][0]) / 1965.0, ((long long)st[k][q][1] - (long long)st[k][0][0]) / 1965.0,
               ((long long)st[k][q][2] - (long long)st[k][0][0]) / 1965.0);
  }
  {
    unsigned long long cs[40][4];
    cudaMemcpyFromSymbol(cs, small_cols, sizeof(cs));
    for (int c = 0; c < 16; ++c)
      printf("col %2d: publish+sync %5lld  rsqrt %5lld  update+shift %5lld  (cycles)  gap-from-prev %5lld\n", c,
             (long long)(cs[c][1] - cs[c][0]), (long long)(cs[c][2] - cs[c][1]), (long long)(cs[c][3] - cs[c][2]),
             c ? (long long)(cs[c][0] - cs[c - 1][3]) : 0ll);
  }
  return 0;
}

// Phase timing of the one-launch 64-wide panel (panel64.cu), standalone: CTA 0 thread 0
// records %globaltimer at each phase boundary (SF_P64_TIMING).  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSF_P64_TIMING -I include \
//        -I paper_1812_02056_b200/csrc calib/p64_probe.cu -o calib/p64_probe
#include <cstdio>
#include <vector>
#include "../paper_1812_02056_b200/csrc/panel64.cu"
namespace sf { void count_launch(int) {} }
int main() {
  using namespace sf;
  const int64_t m = 4096, w = 64;
  std::vector<double> h(m * m);
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < m; ++i) h[i + j * m] = (i == j) ? m : ((i * 7 + j * 13) % 17 - 8) / 17.0;
  double *d, *tol; long long* fail;
  cudaMalloc(&d, m * m * 8); cudaMalloc(&tol, 8); cudaMalloc(&fail, 16);
  const double t0 = 1e-300;
  cudaMemcpy(tol, &t0, 8, cudaMemcpyHostToDevice);
  const char* names[] = {"load D", "sync", "D11", "L21/U12", "D22 upd", "D22", "build M", "last reader", "load x", "subst"};
  for (int rep = 0; rep < 6; ++rep) {
    cudaMemcpy(d, h.data(), m * m * 8, cudaMemcpyHostToDevice);
    long long init[2] = {kNoFail, 0};
    cudaMemcpy(fail, init, 16, cudaMemcpyHostToDevice);
    unsigned long long z[16] = {0};
    z[10] = ~0ull;
    cudaMemcpyToSymbol(p64_times, z, sizeof(z));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    lu_panel64<double>(m, m - w, (int)w, d, m, d, m, 0, tol, fail, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long t[16], tc[16];
    cudaMemcpyFromSymbol(t, p64_times, sizeof(t));
    cudaMemcpyFromSymbol(tc, p64_times_col, sizeof(tc));
    printf("rep %d: %.1f us total;", rep, ms * 1000);
    for (int k = 1; k < 10; ++k) printf(" %s %.2f", names[k], (t[k] - t[k - 1]) / 1000.0);
    printf(" | CTA0 start->T0 %.2f, grid span %.2f, rows done %.2f (us) err=%s\n", (t[0] - t[10]) / 1000.0,
           (t[11] - t[10]) / 1000.0, (t[12] - t[10]) / 1000.0, cudaGetErrorString(cudaGetLastError()));
    printf("   column CTA:");
    for (int k = 1; k < 10; ++k) printf(" %s %.2f", names[k], (tc[k] - tc[k - 1]) / 1000.0);
    printf(" | start->T0 %.2f, done at %.2f (us)\n", (tc[0] - t[10]) / 1000.0, (tc[9] - t[10]) / 1000.0);
  }
  return 0;
}

// Phase cycles of the QR panel kernel (qr_mgs_ll_kernel, SF_MGS_TIMING) at cfg4's panel shape:
// n = 8192, w = 128 (one eager panel through qr_mgs_panel).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSF_MGS_TIMING -I include \
//        -I paper_1812_02056_b200/csrc calib/mgs_ll_probe.cu -o calib/mgs_ll_probe
#include <cstdio>
#include <vector>
#include "../paper_1812_02056_b200/csrc/panels.cu"
namespace sf { void count_launch(int) {} }
int main() {
  using namespace sf;
  const int64_t n = 8192; const int w = 128;
  std::vector<double> h(n * w);
  unsigned s = 12345;
  for (auto& v : h) { s = s * 1664525u + 1013904223u; v = ((s >> 8) & 0xffff) / 65536.0 - 0.5; }
  double *V, *Q, *tol, *work; long long* fail;
  cudaMalloc(&V, n * w * 8); cudaMalloc(&Q, n * w * 8); cudaMalloc(&tol, 8); cudaMalloc(&fail, 16);
  const size_t we = qr_mgs_work_elems(n, w, 8) + 64;
  cudaMalloc(&work, we * 8);
  cudaMemcpy(V, h.data(), n * w * 8, cudaMemcpyHostToDevice);
  const double t0 = 1e-300; cudaMemcpy(tol, &t0, 8, cudaMemcpyHostToDevice);
  const char* names[] = {"cluster bar", "dsmem+put", "ll gather", "gram sum", "scale", "project"};
  for (int rep = 0; rep < 3; ++rep) {
    long long init[2] = {kNoFail, 0};
    cudaMemcpy(fail, init, 16, cudaMemcpyHostToDevice);
    cudaMemset(work, 0, we * 8);
    unsigned long long z[256][8] = {};
    cudaMemcpyToSymbol(mgs_times, z, sizeof(z));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    cudaError_t e = qr_mgs_panel<double>(n, w, V, n, Q, n, 0, tol, work, fail, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long t[256][8];
    cudaMemcpyFromSymbol(t, mgs_times, sizeof(t));
    printf("rep %d: %.1f us (%.2f us/column) (%s / %s)\n", rep, ms * 1000, ms * 1000 / w, cudaGetErrorString(e),
           cudaGetErrorString(cudaGetLastError()));
    for (int g : {0, 7, 63}) {
      printf("  cta %2d:", g);
      for (int p = 0; p < 6; ++p) printf(" %s %.2f", names[p], t[g][p] / 1965.0 / w);
      printf(" (us per column)\n");
    }
  }
  return 0;
}

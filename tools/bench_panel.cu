// Panel Out = Cin + sgn In M at cfg2 shapes (n = 14,287, s = 128): the tiled k_panel (64 x 64 CTAs)
// against the one-wave row-range k_panel_rows, warm (L2 not flushed) and with an L2 flush between
// launches; CUDA-event timing over many launches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bench_panel tools/bench_panel.cu
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_2101_12164_b200/csrc/nsp_blas.cu"
void nsp_count_launch() {}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 14287;
  const int s = 128;
  std::vector<double> h(n * s), hm(s * s);
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  for (auto& v : h) v = nd(g);
  for (auto& v : hm) v = nd(g);
  double *In, *Cin, *Out, *Out2, *M, *flush, *np;
  cudaMalloc(&In, n * s * 8);
  cudaMalloc(&Cin, n * s * 8);
  cudaMalloc(&Out, n * s * 8);
  cudaMalloc(&Out2, n * s * 8);
  cudaMalloc(&M, s * s * 8);
  cudaMalloc(&np, ((n + 63) / 64 + 1) * s * 8);
  const size_t fl = 256ull << 20;
  cudaMalloc(&flush, fl);
  cudaMemcpy(In, h.data(), n * s * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(Cin, h.data(), n * s * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(M, hm.data(), s * s * 8, cudaMemcpyHostToDevice);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](int which, double* out) {
    if (which == 0) {
      PanelArgs a{out, s, Cin, s, In, s, M, s, -1.0, np};
      nspb::panel2(a, nullptr, s, s, n, st);
    } else {
      nspb::panel(out, s, Cin, s, In, s, M, s, s, s, n, -1.0, np, st);
    }
  };
  for (int which = 0; which < 2; ++which)
    for (int cold = 0; cold < 2; ++cold) {
      double* out = which ? Out2 : Out;
      for (int i = 0; i < 5; ++i) run(which, out);
      float tot = 0;
      const int reps = 50;
      for (int i = 0; i < reps; ++i) {
        if (cold) cudaMemsetAsync(flush, i & 0xff, fl, st);
        cudaEventRecord(e0, st);
        run(which, out);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      const double us = tot / reps * 1e3;
      printf("%-12s %-5s %8.2f us  %6.2f TFLOP/s\n", which ? "panel_rows" : "panel_tiled", cold ? "cold" : "warm", us,
             2.0 * n * s * s / (us * 1e-6) / 1e12);
    }
  std::vector<double> a(n * s), b(n * s);
  cudaMemcpy(a.data(), Out, n * s * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), Out2, n * s * 8, cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  for (int64_t i = 0; i < n * s; ++i) {
    md = std::max(md, std::fabs(a[i] - b[i]));
    mx = std::max(mx, std::fabs(a[i]));
  }
  printf("max |tiled - rows| = %.3e (max |out| %.3e)  %s\n", md, mx, cudaGetErrorString(cudaGetLastError()));
  return 0;
}

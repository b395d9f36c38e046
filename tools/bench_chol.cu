#include <cstdio>
#include <vector>
#include <random>
#include <cuda_runtime.h>
struct BcgStatus { int width, indefinite, fallback, converged, nonfinite, pad_[3]; double relres; double scalar[6]; };
template <int STAGE, int RA>
__global__ void __launch_bounds__(32 * 128 / RA) kx_chol(const double* __restrict__ Ain, int sp, int mode, int nact,
                                                     double tau, double* __restrict__ Out, BcgStatus* st) {
  extern __shared__ double sm[];
  const int ld = sp + 1;
  double* Ls = sm;                       // sp x ld
  __shared__ double colv[128];
  __shared__ double xrow[2][128];
  __shared__ double piv[128];
  __shared__ double invd[128];
  __shared__ double sd;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int i0 = RA * ty, j0 = 4 * tx;
  const bool rows_ok = i0 < sp, cols_ok = j0 < sp;
  const int width = nact < 0 ? st->width : nact;
  double r[RA][4];
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + a, j = j0 + b;
      double v = 0.0;
      if (rows_ok && cols_ok) {
        v = Ain[i * sp + j];
        if (i >= width || j >= width) v = (i == j) ? 1.0 : 0.0;
      }
      r[a][b] = v;
    }
  // ---- Cholesky
  bool fail = false;
  for (int c = 0; c < sp; ++c) {
    const int cq = c >> 2, cr = c & 3;
    if (tx == cq && ty == c / RA) {
#pragma unroll
      for (int a = 0; a < RA; ++a)
        if (a == c % RA) sd = r[a][cr];
    }
    __syncthreads();
    const double d = sd;
    if (!(d > 0.0)) {
      fail = true;
      break;
    }
    const double l = sqrt(d);
    const double il = 1.0 / l;
    if (tx == 0 && ty == 0) {
      piv[c] = d;
      invd[c] = il;
    }
    if (tx == cq && i0 + RA - 1 >= c && rows_ok) {
#pragma unroll
      for (int a = 0; a < RA; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if (b == cr) {
            const int i = i0 + a;
            if (i > c) {
              const double v = r[a][b] * il;
              colv[i] = v;
              r[a][b] = v;
            } else if (i == c) {
              r[a][b] = l;
            }
          }
    }
    __syncthreads();
    if (i0 + RA - 1 > c && rows_ok && j0 + 3 > c && cols_ok) {
      double ci[RA], cj[4];
#pragma unroll
      for (int a = 0; a < RA; ++a) ci[a] = colv[min(i0 + a, sp - 1)];
#pragma unroll
      for (int b = 0; b < 4; ++b) cj[b] = colv[min(j0 + b, sp - 1)];
#pragma unroll
      for (int a = 0; a < RA; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = i0 + a, j = j0 + b;
          if (j > c && i >= j) r[a][b] -= ci[a] * cj[b];
        }
    }
  }
  __syncthreads();
  if (STAGE == 0) return;
  if (fail) {
    if (tx == 0 && ty == 0) {
      if (mode == 0) st->indefinite = 1;
      else st->fallback = 1;
    }
    return;
  }
  if (mode == 1) {
    double mn = piv[0], mx = piv[0];
    for (int i = 1; i < width; ++i) {
      mn = fmin(mn, piv[i]);
      mx = fmax(mx, piv[i]);
    }
    if (!(mn > tau * mx)) {
      if (tx == 0 && ty == 0) st->fallback = 1;
      return;
    }
    if (tx == 0 && ty == 0) {
      st->fallback = 0;
      st->width = width;
    }
  }
  if (STAGE == 1) return;
  // ---- L to smem (lower), X = L^{-1} in registers
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = i0 + a, j = j0 + b;
      if (rows_ok && cols_ok) Ls[i * ld + j] = (j <= i) ? r[a][b] : 0.0;
      r[a][b] = (rows_ok && cols_ok && i == j) ? 1.0 : 0.0;
    }
  __syncthreads();
  for (int k = 0; k < sp; ++k) {
    const int kq = k / RA, kr = k % RA;
    double* xr = xrow[k & 1];
    if (ty == kq && cols_ok) {
      const double ilkk = invd[k];
#pragma unroll
      for (int a = 0; a < RA; ++a)
        if (a == kr)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int j = j0 + b;
            if (j <= k) r[a][b] *= ilkk;
            xr[j] = r[a][b];
          }
    }
    __syncthreads();
    if (i0 + RA - 1 > k && rows_ok && j0 <= k && cols_ok) {
      double li[RA], xj[4];
#pragma unroll
      for (int a = 0; a < RA; ++a) li[a] = Ls[min(i0 + a, sp - 1) * ld + k];
#pragma unroll
      for (int b = 0; b < 4; ++b) xj[b] = xr[j0 + b];
#pragma unroll
      for (int a = 0; a < RA; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = i0 + a, j = j0 + b;
          if (i > k && j <= k) r[a][b] -= li[a] * xj[b];
        }
    }
  }
  __syncthreads();
  if (mode == 1) {
    if (rows_ok && cols_ok)
#pragma unroll
      for (int a = 0; a < RA; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) Out[(j0 + b) * sp + i0 + a] = r[a][b];  // T = X^T
    return;
  }
  // mode 0: D^{-1} = X^T X (X lower triangular)
  if (rows_ok && cols_ok)
#pragma unroll
    for (int a = 0; a < RA; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) Ls[(i0 + a) * ld + j0 + b] = r[a][b];
  __syncthreads();
  if (!(rows_ok && cols_ok)) return;
  double acc[RA][4];
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k = max(i0, j0); k < sp; ++k) {
    double xi[RA], xj[4];
#pragma unroll
    for (int a = 0; a < RA; ++a) xi[a] = Ls[k * ld + i0 + a];
#pragma unroll
    for (int b = 0; b < 4; ++b) xj[b] = Ls[k * ld + j0 + b];
#pragma unroll
    for (int a = 0; a < RA; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = fma(xi[a], xj[b], acc[a][b]);
  }
#pragma unroll
  for (int a = 0; a < RA; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) Out[(i0 + a) * sp + j0 + b] = acc[a][b];
}


int main() {
  const int sp = 128;
  std::vector<double> G(sp*sp);
  std::mt19937_64 g(1); std::normal_distribution<double> nd;
  std::vector<double> W(1000*sp); for (auto& x: W) x = nd(g);
  for (int i=0;i<sp;++i) for (int j=0;j<sp;++j){double s=0; for(int r=0;r<1000;++r) s+=W[r*sp+i]*W[r*sp+j]; G[i*sp+j]=s;}
  double *dG,*dO; BcgStatus* st; cudaMalloc(&dG,sp*sp*8); cudaMalloc(&dO,sp*sp*8); cudaMalloc(&st,sizeof(BcgStatus));
  cudaMemcpy(dG,G.data(),sp*sp*8,cudaMemcpyHostToDevice);
  BcgStatus h{}; h.width=sp; cudaMemcpy(st,&h,sizeof(h),cudaMemcpyHostToDevice);
  size_t smem=(size_t)sp*(sp+1)*8;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  auto run=[&](const char* nm, auto f){ for(int i=0;i<3;++i) f(); cudaEventRecord(e0); for(int i=0;i<10;++i) f(); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); printf("%s %.2f us %s\n",nm,ms*100,cudaGetErrorString(cudaGetLastError()));};
#define RUN(ST, RA, MODE, NACT) cudaFuncSetAttribute(kx_chol<ST,RA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
  run("stage " #ST " RA " #RA " mode " #MODE, [&]{kx_chol<ST,RA><<<1,dim3(32,128/RA),smem>>>(dG,sp,MODE,NACT,1e-14,dO,st);});
  RUN(0,4,1,sp) RUN(0,8,1,sp) RUN(0,16,1,sp)
  RUN(2,4,1,sp) RUN(2,8,1,sp) RUN(2,16,1,sp)
  RUN(2,4,0,-1) RUN(2,8,0,-1) RUN(2,16,0,-1)
  return 0;
}

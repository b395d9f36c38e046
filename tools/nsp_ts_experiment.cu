// EXPERIMENT (not built into libnsp): 148-SM-balanced tall-skinny kernels; measured slower than the
// nsp_blas.cu kernels at s = 128 (tools/bench_ts.cu, round 1) - kept for the next tuning pass.
// Tall-skinny fp64 contractions of the block-CG iteration on the DMMA pipe (§8(a) rows a6, a8, a10,
// a11; north_star (c) "Gram products as tall-skinny fp64 contractions on the DMMA tensor pipe"),
// sized to the 148 SMs so that no wave is left mostly empty:
//  k_ts_gram   out = Xa^T Xb (n x sa)^T (n x sb), sa, sb in {64, 128}: one CTA per SM, each over a
//              CONTIGUOUS row range (n/148 rows, any remainder handled by a short final k-loop so
//              every SM does the same work), 8 warps each owning a (sa/4) x (sb/2) output block in
//              registers; 32-row K slabs double-buffered with cp.async; per-CTA partials reduced in
//              a fixed order (deterministic, reading C17).  sym: only the lower output blocks are
//              computed and mirrored (W^T W).
//  k_ts_panel  Out = Cin + sgn * In M (n x kdim times kdim x ncols, ncols in {64, 128}), optionally
//              two argument sets sharing M (X += P alpha, R -= Q alpha): M staged once per CTA in
//              shared memory; warps stream 8-row slabs (1786 slabs for n = 14,287 -> 12-13 per SM)
//              with the A fragments loaded straight from global (L2) and the column sums of
//              squares of the output (R's norms, a8) reduced per slab in registers.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "../paper_2101_12164_b200/csrc/nsp_blas.h"
#include "../paper_2101_12164_b200/csrc/nsp_dmma.cuh"

using namespace nspd;

namespace {

constexpr int TS_SMS = 148;
constexpr int KS = 32;        // K-slab rows of the Gram

__device__ __forceinline__ void cp16_zf(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

// rows x cols (cols even) from row-major global (ld gld) to smem (ld sld); rows >= nvalid zero
__device__ __forceinline__ void stage(double* s, int sld, const double* g, int64_t gld, int rows, int cols,
                                      int64_t nvalid) {
  const int cpr = cols / 2;
  for (int c = threadIdx.x; c < rows * cpr; c += blockDim.x) {
    const int r = c / cpr, q = c - r * cpr;
    const bool v = r < nvalid;
    cp16_zf(s + r * sld + 2 * q, v ? (const void*)(g + r * gld + 2 * q) : (const void*)g, v);
  }
}

// MF m-fragments (8 rows of the output = 8 columns of Xa) x NF n-fragments per warp
template <int MF, int NF>
__global__ void __launch_bounds__(256) k_ts_gram(const double* __restrict__ Xa, int lda, const double* __restrict__ Xb,
                                                 const double* __restrict__ Xb2, int ldb, int64_t n, int sym,
                                                 double* __restrict__ part) {
  constexpr int SA = 4 * 8 * MF, SB = 2 * 8 * NF;   // output sa x sb per Xb
  constexpr int LD = (SA > SB ? SA : SB) + 8;       // == 8 mod 32 doubles: conflict-free fragments
  extern __shared__ double sm[];
  double* As[2] = {sm, sm + KS * LD};
  double* Bs[2] = {sm + 2 * KS * LD, sm + 3 * KS * LD};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int mb = warp >> 1, nb = warp & 1;
  const double* B = blockIdx.y ? Xb2 : Xb;
  const int64_t r0 = n * blockIdx.x / gridDim.x, r1 = n * (blockIdx.x + 1) / gridDim.x;
  const bool active = !(sym && (8 * MF * mb + 8 * MF - 1 < 8 * NF * nb));   // upper block of a symmetric Gram
  double acc[MF][NF][2];
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  int buf = 0;
  if (r0 < r1) {
    stage(As[0], LD, Xa + r0 * lda, lda, KS, SA, r1 - r0);
    stage(Bs[0], LD, B + r0 * ldb, ldb, KS, SB, r1 - r0);
    cp_commit();
  }
  for (int64_t r = r0; r < r1; r += KS) {
    const int64_t rn = r + KS;
    if (rn < r1) {
      stage(As[buf ^ 1], LD, Xa + rn * lda, lda, KS, SA, r1 - rn);
      stage(Bs[buf ^ 1], LD, B + rn * ldb, ldb, KS, SB, r1 - rn);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const int64_t krem = ((r1 - r + 3) / 4) * 4;
    const int kmax = krem < KS ? (int)krem : KS;   // short final slab
    if (active) {
      const double* A = As[buf];
      const double* Bm = Bs[buf];
#pragma unroll 2
      for (int k = 0; k < kmax; k += 4) {
        double a[MF], b[NF];
#pragma unroll
        for (int i = 0; i < MF; ++i) a[i] = A[(k + t) * LD + 8 * MF * mb + 8 * i + g];
#pragma unroll
        for (int j = 0; j < NF; ++j) b[j] = Bm[(k + t) * LD + 8 * NF * nb + 8 * j + g];
#pragma unroll
        for (int i = 0; i < MF; ++i)
#pragma unroll
          for (int j = 0; j < NF; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
    __syncthreads();
    buf ^= 1;
  }
  double* out = part + ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * (SA * SB);
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int rr = 8 * MF * mb + 8 * i + g, cc = 8 * NF * nb + 8 * j + 2 * t;
      *reinterpret_cast<double2*>(out + rr * SB + cc) =
          active ? make_double2(acc[i][j][0], acc[i][j][1]) : make_double2(0.0, 0.0);
    }
}

// out[y][i][j] = sum_c part[y][c][i][j] in fixed order (4 interleaved groups combined in order);
// sym: the upper triangle mirrors the lower.
__global__ void k_ts_gram_reduce(const double* __restrict__ part, int nparts, int sa, int sb, int sym,
                                 double* __restrict__ out, double* __restrict__ out2, int ldo) {
  __shared__ double red[4][64];
  const int e = blockIdx.x * 64 + threadIdx.x;
  const int y = blockIdx.y;
  const int g = threadIdx.y;
  const int i = e / sb, j = e - i * sb;
  const bool valid = e < sa * sb;
  const int src = (sym && j > i) ? j * sb + i : e;
  double s = 0.0;
  if (valid) {
    const double* p = part + (int64_t)y * nparts * sa * sb + src;
    for (int c = g; c < nparts; c += 4) s += p[(int64_t)c * sa * sb];
  }
  red[g][threadIdx.x] = s;
  __syncthreads();
  if (g == 0 && valid) {
    const double v = (red[0][threadIdx.x] + red[1][threadIdx.x]) + (red[2][threadIdx.x] + red[3][threadIdx.x]);
    (y ? out2 : out)[(int64_t)i * ldo + j] = v;
  }
}

struct TsArgs {
  double* Out;
  int ldo;
  const double* Cin;
  int ldc;
  const double* In;
  int ldi;
  double sgn;
  double* normpart;   // [slab][ncols] column sums of squares of Out, or null
};

template <int NF>
__global__ void __launch_bounds__(256) k_ts_panel(TsArgs a0, TsArgs a1, int nz, const double* __restrict__ M, int ldm,
                                                  int kdim, int64_t n) {
  constexpr int NC = 8 * NF;
  constexpr int LDM = NC + 8;
  extern __shared__ double Ms[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  {
    const int cpr = NC / 2;
    for (int c = tid; c < kdim * cpr; c += 256) {
      const int r = c / cpr, q = c - r * cpr;
      cp_async16(Ms + r * LDM + 2 * q, M + (int64_t)r * ldm + 2 * q);
    }
    cp_commit();
    cp_wait<0>();
    __syncthreads();
  }
  const int64_t nslab = (n + 7) / 8;
  const int64_t total = nslab * nz;
  // contiguous slab range per CTA (equal work per SM), warps round-robin inside it
  const int64_t s0 = total * blockIdx.x / gridDim.x, s1 = total * (blockIdx.x + 1) / gridDim.x;
  for (int64_t sidx = s0 + warp; sidx < s1; sidx += 8) {
    const int z = (int)(sidx % nz);
    const int64_t slab = sidx / nz;
    const TsArgs& p = z ? a1 : a0;
    const int64_t row = slab * 8 + g;
    const bool rv = row < n;
    const double* in = p.In + (rv ? row : 0) * (int64_t)p.ldi;
    double acc[NF][2];
#pragma unroll
    for (int j = 0; j < NF; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll 4
    for (int k = 0; k < kdim; k += 4) {
      const double a = rv ? __ldg(in + k + t) : 0.0;
#pragma unroll
      for (int j = 0; j < NF; ++j) dmma(acc[j][0], acc[j][1], a, Ms[(k + t) * LDM + 8 * j + g]);
    }
    double sq[NF][2];
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      const int c = 8 * j + 2 * t;
      double v0 = p.sgn * acc[j][0], v1 = p.sgn * acc[j][1];
      if (rv) {
        if (p.Cin) {
          const double2 cv = *reinterpret_cast<const double2*>(p.Cin + row * p.ldc + c);
          v0 += cv.x;
          v1 += cv.y;
        }
        *reinterpret_cast<double2*>(p.Out + row * p.ldo + c) = make_double2(v0, v1);
      } else {
        v0 = v1 = 0.0;
      }
      sq[j][0] = v0 * v0;
      sq[j][1] = v1 * v1;
    }
    if (p.normpart) {   // column sums over the slab's 8 rows (lanes g), fixed butterfly order
#pragma unroll
      for (int j = 0; j < NF; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double v = sq[j][e];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          sq[j][e] = v;
        }
      if (g == 0)
#pragma unroll
        for (int j = 0; j < NF; ++j)
          *reinterpret_cast<double2*>(p.normpart + slab * NC + 8 * j + 2 * t) = make_double2(sq[j][0], sq[j][1]);
    }
  }
}

}  // namespace

namespace nspb {

size_t ts_gram_ws_doubles(int sa, int sb) { return (size_t)2 * TS_SMS * sa * sb; }

static void ts_gram_launch(const double* Xa, int lda, int sa, const double* Xb, const double* Xb2, int ldb, int sb,
                           int64_t n, bool sym, double* out, double* out2, int ldo, double* ws, cudaStream_t st) {
  const int ny = Xb2 ? 2 : 1;
  const dim3 grid(TS_SMS, ny);
#define NSP_TS_GRAM(MF, NF)                                                                          \
  {                                                                                                  \
    constexpr int LD = ((32 * MF > 16 * NF) ? 32 * MF : 16 * NF) + 8;                                \
    const size_t smem = 4 * KS * LD * sizeof(double);                                                \
    static bool attr = false;                                                                        \
    if (!attr) {                                                                                     \
      cudaFuncSetAttribute(k_ts_gram<MF, NF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      attr = true;                                                                                   \
    }                                                                                                \
    nsp_count_launch();                                                                              \
    k_ts_gram<MF, NF><<<grid, 256, smem, st>>>(Xa, lda, Xb, Xb2, ldb, n, sym ? 1 : 0, ws);          \
  }
  if (sa == 128 && sb == 128) NSP_TS_GRAM(4, 8)
  else if (sa == 128 && sb == 64) NSP_TS_GRAM(4, 4)
  else if (sa == 64 && sb == 128) NSP_TS_GRAM(2, 8)
  else NSP_TS_GRAM(2, 4)
#undef NSP_TS_GRAM
  nsp_count_launch();
  k_ts_gram_reduce<<<dim3((sa * sb + 63) / 64, ny), dim3(64, 4), 0, st>>>(ws, TS_SMS, sa, sb, sym ? 1 : 0, out,
                                                                          out2, ldo);
}

void ts_gram(const double* Xa, int lda, int sa, const double* Xb, int ldb, int sb, int64_t n, bool sym, double* out,
             int ldo, double* ws, cudaStream_t st) {
  ts_gram_launch(Xa, lda, sa, Xb, nullptr, ldb, sb, n, sym, out, nullptr, ldo, ws, st);
}

void ts_gram2(const double* Xa, int lda, int sa, const double* Xb, const double* Xb2, int ldb, int sb, int64_t n,
              double* out, double* out2, int ldo, double* ws, cudaStream_t st) {
  ts_gram_launch(Xa, lda, sa, Xb, Xb2, ldb, sb, n, false, out, out2, ldo, ws, st);
}

void ts_panel2(const PanelArgs& a0, const PanelArgs* a1, int kdim, int ncols, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  TsArgs t0{a0.Out, a0.ldo, a0.Cin, a0.ldc, a0.In, a0.ldi, a0.sgn, a0.normpart};
  TsArgs t1 = t0;
  if (a1) t1 = TsArgs{a1->Out, a1->ldo, a1->Cin, a1->ldc, a1->In, a1->ldi, a1->sgn, a1->normpart};
  const int nz = a1 ? 2 : 1;
  const int64_t slabs = ((n + 7) / 8) * nz;
  const unsigned grid = (unsigned)std::min<int64_t>(TS_SMS, (slabs + 7) / 8);
  if (ncols == 128) {
    const size_t smem = (size_t)kdim * (128 + 8) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_ts_panel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(128 * 136 * 8));
      attr = true;
    }
    nsp_count_launch();
    k_ts_panel<16><<<grid, 256, smem, st>>>(t0, t1, nz, a0.M, a0.ldm, kdim, n);
  } else {
    const size_t smem = (size_t)kdim * (64 + 8) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_ts_panel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(128 * 72 * 8));
      attr = true;
    }
    nsp_count_launch();
    k_ts_panel<8><<<grid, 256, smem, st>>>(t0, t1, nz, a0.M, a0.ldm, kdim, n);
  }
}

}  // namespace nspb

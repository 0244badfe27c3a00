// Compressed M2L on the device (M2LOperatorSet, m2l.cpp:12-204; bench.cpp:288-299).
//
// Precompute (once per context): the 16 canonical operators are assembled at unit
// width (m2l.cpp:90-111) and compressed with a truncated SVD on the device
// (cuSOLVER dgesvd, rank rule of m2l.cpp:116-122), or loaded from the reference's
// binary cache (m2l.cpp:247-288). Each admissible transfer vector v (316) gets the
// permuted factors of its class: since the reference applies
//     local[t][m] += scale * sum_k U[p_v[m]][k] * sigma_k * sum_n V[p_v[n]][k] * W[s][n]
// (gather z[p[n]] = W[n], Y = U sigma V^T z, scatter out[m] += scale y[p[m]],
// m2l.cpp:189-203), the per-vector operator is M2_v M1_v with
//     M1_v[k][n] = sigma_k V[p_v[n]][k]   (r x l^3)
//     M2_v[m][k] = U[p_v[m]][k]           (l^3 x r).
//
// Evaluation per level as two dense FP64 GEMMs per parity class (DESIGN.md
// "M2L as two GEMMs"). The admissible vectors of a target depend only on the parity
// of its grid coordinates (an axis component of +3 needs an even target, -3 an odd
// one), so for each of the 8 parity classes:
//   phase A  Y = M1_p (R x l^3) * W (l^3 x sources of parity p), M1_p the stack of
//            M1_v over the 189 vectors admissible from a parity-p source; the
//            epilogue scatters block v of source s to target s - v (if it exists)
//            into Yt[t] (target-side stacking order);
//   phase B  local_own[t] += scale * M2_q (l^3 x R) * Yt[t] for targets of parity q
//            (= instead of += inside an evaluation).
//            Yt is one array per level, zeroed once at allocation (and kept across
//            tree rebuilds for full levels); the blocks of absent sources t + v are
//            never written, so they stay exactly zero.
// Same arithmetic as the reference (4 l^3 r per pair), on DMMA (mma.sync
// m8n8k4 f64, the B200 FP64 tensor path: 37.2 TF/s measured, profiles/r01_fp64_peaks.txt).
#include <cusolverDn.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace fmmgpu {

// ------------------------------------------------------------------ symmetry tables
// cube_symmetries (m2l.cpp:12-25): perm-major, sign bit of axis a = bit (2-a).
int canonicalize_host(const int v[3], int perm_out[3], int sign_out[3]) {
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  const int d = std::max({std::abs(v[0]), std::abs(v[1]), std::abs(v[2])});
  if (d < 2 || d > 3) throw Error(FMMGPU_INVALID_ARGUMENT, "canonicalize_m2l_vector: max-norm must be 2 or 3");
  for (const auto& p : perms)
    for (int bits = 0; bits < 8; ++bits) {
      int sign[3], u[3];
      for (int a = 0; a < 3; ++a) {
        sign[a] = (bits >> (2 - a)) & 1 ? -1 : 1;
        u[a] = sign[a] * v[p[a]];
      }
      if (!(u[0] >= u[1] && u[1] >= u[2] && u[2] >= 0 && u[0] >= 2 && u[0] <= 3)) continue;
      // canonical list (m2l.cpp:45-55): i = 2..3, j = 0..i, k = 0..j
      int idx = 0;
      for (int i = 2; i <= 3; ++i)
        for (int j = 0; j <= i; ++j)
          for (int k = 0; k <= j; ++k, ++idx)
            if (u[0] == i && u[1] == j && u[2] == k) {
              for (int a = 0; a < 3; ++a) {
                perm_out[a] = p[a];
                sign_out[a] = sign[a];
              }
              return idx;
            }
    }
  throw Error(FMMGPU_LOGIC_ERROR, "canonicalize_m2l_vector: no symmetry found");
}

namespace {

void canonical_vector(int c, int out[3]) {
  int idx = 0;
  for (int i = 2; i <= 3; ++i)
    for (int j = 0; j <= i; ++j)
      for (int k = 0; k <= j; ++k, ++idx)
        if (idx == c) { out[0] = i; out[1] = j; out[2] = k; return; }
}

// grid_permutation (m2l.cpp:72-88): p[flat(m)] = flat(g m)
std::vector<uint32_t> grid_perm(const int perm[3], const int sign[3], int l) {
  std::vector<uint32_t> p(size_t(l) * l * l);
  int m[3];
  for (m[0] = 0; m[0] < l; ++m[0])
    for (m[1] = 0; m[1] < l; ++m[1])
      for (m[2] = 0; m[2] < l; ++m[2]) {
        uint32_t flat = 0;
        for (int a = 0; a < 3; ++a) {
          const int cc = sign[a] > 0 ? m[perm[a]] : l - 1 - m[perm[a]];
          flat = flat * l + cc;
        }
        p[(m[0] * l + m[1]) * l + m[2]] = flat;
      }
  return p;
}

void slot_vec(int slot, int v[3]) {
  v[0] = slot / 49 - 3;
  v[1] = (slot / 7) % 7 - 3;
  v[2] = slot % 7 - 3;
}

// admissible for a target of parity q (bit 2 = i, bit 1 = j, bit 0 = k, the Morton
// octant): max-norm 2..3 and +3 needs an even, -3 an odd target coordinate
// (parents adjacent, geometry.cpp:255-275).
bool admissible_for_target(const int v[3], int q) {
  if (std::max({std::abs(v[0]), std::abs(v[1]), std::abs(v[2])}) < 2) return false;
  for (int a = 0; a < 3; ++a) {
    const int qa = (q >> (2 - a)) & 1;
    if (v[a] == 3 && qa != 0) return false;
    if (v[a] == -3 && qa != 1) return false;
  }
  return true;
}
int vec_parity(const int v[3]) { return ((v[0] & 1) << 2) | ((v[1] & 1) << 1) | (v[2] & 1); }

#define CUSOLVER_CHECK(x)                                                                     \
  do {                                                                                        \
    cusolverStatus_t st_ = (x);                                                               \
    if (st_ != CUSOLVER_STATUS_SUCCESS)                                                       \
      throw Error(FMMGPU_RUNTIME_ERROR, "cuSOLVER error " + std::to_string(int(st_)) + " at " + \
                                            std::to_string(__LINE__));                        \
  } while (0)

// assemble_m2l (m2l.cpp:90-111) at unit width + truncated SVD on the device
void compute_factors(fmmgpu_ctx* c) {
  const int l = c->order, n3 = c->l3;
  std::vector<double> nodes(3 * n3);
  for (int a = 0, idx = 0; a < l; ++a)
    for (int b = 0; b < l; ++b)
      for (int cc = 0; cc < l; ++cc, ++idx) {
        nodes[3 * idx] = c->h_roots[a] * 0.5 * 1.0;
        nodes[3 * idx + 1] = c->h_roots[b] * 0.5 * 1.0;
        nodes[3 * idx + 2] = c->h_roots[cc] * 0.5 * 1.0;
      }
  cusolverDnHandle_t h;
  CUSOLVER_CHECK(cusolverDnCreate(&h));
  double *dA, *dS, *dU, *dVT, *dWork, *dRW;
  int* dInfo;
  int lwork = 0;
  FMM_CUDA(cudaMalloc(&dA, sizeof(double) * n3 * n3));
  FMM_CUDA(cudaMalloc(&dU, sizeof(double) * n3 * n3));
  FMM_CUDA(cudaMalloc(&dVT, sizeof(double) * n3 * n3));
  FMM_CUDA(cudaMalloc(&dS, sizeof(double) * n3));
  FMM_CUDA(cudaMalloc(&dRW, sizeof(double) * n3));
  FMM_CUDA(cudaMalloc(&dInfo, sizeof(int)));
  CUSOLVER_CHECK(cusolverDnDgesvd_bufferSize(h, n3, n3, &lwork));
  FMM_CUDA(cudaMalloc(&dWork, sizeof(double) * lwork));
  std::vector<double> K(size_t(n3) * n3), U(size_t(n3) * n3), VT(size_t(n3) * n3), S(n3);
  for (int cl = 0; cl < 16; ++cl) {
    int v[3];
    canonical_vector(cl, v);
    for (int m = 0; m < n3; ++m)
      for (int n = 0; n < n3; ++n) {
        const double dx = nodes[3 * m] - v[0] * 1.0 - nodes[3 * n];
        const double dy = nodes[3 * m + 1] - v[1] * 1.0 - nodes[3 * n + 1];
        const double dz = nodes[3 * m + 2] - v[2] * 1.0 - nodes[3 * n + 2];
        K[size_t(n) * n3 + m] = 1.0 / std::sqrt(dx * dx + dy * dy + dz * dz);  // column-major
      }
    FMM_CUDA(cudaMemcpy(dA, K.data(), sizeof(double) * K.size(), cudaMemcpyHostToDevice));
    CUSOLVER_CHECK(cusolverDnDgesvd(h, 'S', 'S', n3, n3, dA, n3, dS, dU, n3, dVT, n3, dWork, lwork, dRW, dInfo));
    int info = 0;
    FMM_CUDA(cudaMemcpy(&info, dInfo, sizeof(int), cudaMemcpyDeviceToHost));
    if (info != 0) throw Error(FMMGPU_RUNTIME_ERROR, "cuSOLVER dgesvd did not converge");
    FMM_CUDA(cudaMemcpy(U.data(), dU, sizeof(double) * U.size(), cudaMemcpyDeviceToHost));
    FMM_CUDA(cudaMemcpy(VT.data(), dVT, sizeof(double) * VT.size(), cudaMemcpyDeviceToHost));
    FMM_CUDA(cudaMemcpy(S.data(), dS, sizeof(double) * S.size(), cudaMemcpyDeviceToHost));
    int r = n3;  // m2l.cpp:116-122
    for (int i = 1; i < n3; ++i)
      if (S[i] <= c->eps * S[0]) {
        r = i;
        break;
      }
    auto& T = c->m2l;
    T.rank[cl] = r;
    T.u[cl].assign(size_t(n3) * r, 0.0);
    T.v[cl].assign(size_t(n3) * r, 0.0);
    T.sigma[cl].assign(S.begin(), S.begin() + r);
    for (int i = 0; i < n3; ++i)
      for (int k = 0; k < r; ++k) {
        T.u[cl][size_t(i) * r + k] = U[size_t(k) * n3 + i];
        T.v[cl][size_t(i) * r + k] = VT[size_t(i) * n3 + k];
      }
  }
  cudaFree(dA); cudaFree(dU); cudaFree(dVT); cudaFree(dS); cudaFree(dRW); cudaFree(dInfo); cudaFree(dWork);
  cusolverDnDestroy(h);
}

// ------------------------------------------------------------------ GEMM kernels

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp16z(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp8z(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

struct GemmArgs {
  LevelView lv;
  const uint32_t* cls_cells;
  uint32_t cls_off[9];
  const double* A;        // [8][rows][lda]
  size_t a_class_stride;  // rows * lda
  int lda;
  int K;                  // multiple of BK
  const double* W;        // phase A: multipoles (ldE)
  int ldE;
  double* Yt;             // [cells][ldY]
  int ldY;
  const int4* rowA;       // phase A epilogue table [8][rowsA]
  const int* tileVec;     // phase A: vector slots per M-tile [8][rowsA/64][vtMax]
  int vtMax;
  int rowsA;
  const int* kslot;       // vector slot per target-stack column [8][ldY] (host tables)
  double* local;          // phase B output (local_own)
  const int* tileVec2;    // streamed phase A: vector slots per 128-row tile [8][rowsA/128][vtMax2]
  int vtMax2;
  int ksplit;             // phase B split-K factor (1 = accumulate directly)
  int rowB0;              // phase B: first row of this launch's M-tiles (tail launches)
  int msplit;             // phase A M-split factor (coarse levels)
  int cls_fast;           // phase A grid: parity class in blockIdx.x (else blockIdx.y)
  int ow;                 // phase B: write local_own instead of accumulating (evaluation)
  double* part;           // phase B split-K partials [ksplit][ncells][ldE]
  uint32_t ncells;
  int l3;
  double scale;
};

// Phase B: local_own[t] += scale * M2_q (rowsB x ldY) * Yt[t] for the targets t of
// parity class q. Optional deterministic split-K for levels too small to fill the
// GPU: split s writes its partial sums to part[s][t][row] and k_m2l_splitk_reduce
// adds them in split order.
template <int BM, int BN, int WM, int WN, int STAGES, int BK>
__global__ void __launch_bounds__(WM* WN * 32) k_m2l_phase_b(const GemmArgs g) {
  constexpr int T = WM * WN * 32;
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int MT = WTM / 8, NT = WTN / 8;
  constexpr int SPAD = BK + 4;  // == 4 (mod 16): conflict-free fragment loads
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                              // [STAGES][BM][SPAD]
  double* Bs = smem + STAGES * BM * SPAD;         // [STAGES][BN][SPAD]
  __shared__ uint32_t col_cell[BN];

  const int cls = blockIdx.z / g.ksplit, split = blockIdx.z % g.ksplit;
  const uint32_t ncls = g.cls_off[cls + 1] - g.cls_off[cls];
  const uint32_t n0 = blockIdx.y * BN;
  if (n0 >= ncls) return;
  const int m0 = g.rowB0 + blockIdx.x * BM;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp / WN, wn = warp % WN;
  const int gq = lane >> 2, tq = lane & 3;

  for (int j = tid; j < BN; j += T) col_cell[j] = (n0 + j < ncls) ? g.cls_cells[g.cls_off[cls] + n0 + j] : NPOS;
  __syncthreads();

  const double* A = g.A + cls * g.a_class_stride + size_t(m0) * g.lda;
  const int KTALL = g.K / BK;
  const int per = (KTALL + g.ksplit - 1) / g.ksplit;
  const int kt0 = split * per;
  const int KT = max(0, min(KTALL, kt0 + per) - kt0);

  auto load_tile = [&](int stage, int kt) {
    const int k0 = (kt0 + kt) * BK;
    double* as = As + stage * BM * SPAD;
    double* bs = Bs + stage * BN * SPAD;
    for (int ch = tid; ch < BM * (BK / 2); ch += T) {
      const int r = ch / (BK / 2), q = (ch % (BK / 2)) * 2;
      cp16(as + r * SPAD + q, A + size_t(r) * g.lda + k0 + q);
    }
    // Yt blocks of absent sources were never written by phase A and stay zero from
    // the allocation (one Yt per level), so the operand is a plain copy. (Resolving the
    // thread's column row pointers once per CTA instead of per slice: 98 -> 128 registers,
    // config-B M2L 12.28 -> 12.34 ms, C 56.94 -> 57.20 ms; tools/gpu/gpu_r02ba.sh.)
    for (int ch = tid; ch < BN * (BK / 2); ch += T) {
      const int j = ch / (BK / 2), q = (ch % (BK / 2)) * 2;
      const uint32_t cell = col_cell[j];
      const bool ok = cell != NPOS;
      cp16z(bs + j * SPAD + q, g.Yt + (ok ? size_t(cell) * g.ldY + k0 + q : 0), ok);
    }
  };

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < KT) load_tile(st, st);
    cp_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int pf = kt + STAGES - 1;
    if (pf < KT) load_tile(pf % STAGES, pf);
    cp_commit();
    const double* as = As + (kt % STAGES) * BM * SPAD + (wm * WTM + gq) * SPAD + tq;
    const double* bs = Bs + (kt % STAGES) * BN * SPAD + (wn * WTN + gq) * SPAD + tq;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = as[i * 8 * SPAD + kk];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = bs[j * 8 * SPAD + kk];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_wait<0>();

  // epilogue: thread holds C[row = gq + 8i][col = 2 tq + e + 8j] of its warp tile
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    const int row = m0 + wm * WTM + i * 8 + gq;
    if (row >= g.l3) continue;
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = wn * WTN + j * 8 + 2 * tq + e;
        const uint32_t t = col_cell[col];
        if (t == NPOS) continue;
        if (g.ksplit == 1) {
          double* out = g.local + size_t(t) * g.ldE + row;
          *out = g.ow ? g.scale * acc[i][j][e] : *out + g.scale * acc[i][j][e];
        } else {
          g.part[(size_t(split) * g.ncells + t) * g.ldE + row] = acc[i][j][e];
        }
      }
  }
}

// over the targets of the phase B list only (the partials of other cells are unset)
__global__ void k_m2l_splitk_reduce(const double* __restrict__ part, int ksplit, uint32_t ncells, int ldE, int l3,
                                    double scale, const uint32_t* __restrict__ targets, uint32_t ntargets,
                                    double* __restrict__ local, int ow) {
  const uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (e >= uint64_t(ntargets) * ldE) return;
  const int row = static_cast<int>(e % ldE);
  if (row >= l3) return;
  const uint64_t i = uint64_t(targets[e / ldE]) * ldE + row;
  double s = part[i];
  for (int k = 1; k < ksplit; ++k) s += part[k * uint64_t(ncells) * ldE + i];
  local[i] = ow ? scale * s : local[i] + scale * s;
}

// Phase A, W-resident: one CTA owns BN source columns of one parity class. Their
// multipoles (BN x K) are staged ONCE in shared memory and the whole stacked operator
// M1_p (R rows) streams past them in BM x BK slices through a cp.async ring that
// runs across M-tile boundaries, so the scatter epilogue of one M-tile overlaps the
// loads of the next and no CTA pays a pipeline ramp per 64 x 64 tile.
// Used for l <= 5: 64-row M-tiles, 2-stage ring of 32-wide k-slices, 64 resident columns
// (W 68 KB + ring 37 KB). Above order 5 the multipoles no longer fit 64 per CTA (24 at
// l = 7), the operator then feeds too few columns per load, and k_m2l_phase_a2 (both
// operands streamed, 128 x 64 tiles) is used instead.
template <int PA_BM, int PA_ST, int BN, int WM, int WN, int PA_BK = 16, int MINB = 2>
__global__ void __launch_bounds__(WM * WN * 32, MINB) k_m2l_phase_a(const GemmArgs g) {
  constexpr int PA_THREADS = WM * WN * 32;
  constexpr int PA_SPAD = PA_BK + 4;  // == 4 (mod 16): conflict-free fragments
  constexpr int WTM = PA_BM / WM, WTN = BN / WN;
  constexpr int MT = WTM / 8, NT = WTN / 8;
  extern __shared__ __align__(16) double smem[];
  const int wpad = g.K + 4;                       // == 4 (mod 16): conflict-free fragments
  double* Ws = smem;                              // [BN][wpad]
  double* As = smem + BN * wpad;                  // [PA_ST][PA_BM][PA_SPAD]
  // [vtMax][BN] target cell of (vector of the M-tile, column): filled at k-slice KT/2 of a
  // tile, read by its epilogue; a __syncthreads separates that epilogue from the next fill
  uint32_t* tgt = reinterpret_cast<uint32_t*>(As + PA_ST * PA_BM * PA_SPAD);
  __shared__ uint32_t col_cell[BN];
  __shared__ int col_ijk[BN][3];

  // class-fastest CTA order (g.cls_fast): the 8 parity classes of one spatial block run
  // back to back, so the neighbouring blocks of a target's Yt row (written by sources of
  // different parities) are completed while their sectors are still in L2
  const int cls = g.cls_fast ? blockIdx.x : blockIdx.y;
  const uint32_t ncls = g.cls_off[cls + 1] - g.cls_off[cls];
  const uint32_t n0 = (g.cls_fast ? blockIdx.y : blockIdx.x) * BN;
  if (n0 >= ncls) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp / WN, wn = warp % WN;
  const int gq = lane >> 2, tq = lane & 3;

  for (int j = tid; j < BN; j += PA_THREADS) {
    const uint32_t cell = (n0 + j < ncls) ? g.cls_cells[g.cls_off[cls] + n0 + j] : NPOS;
    col_cell[j] = cell;
    int ijk[3] = {0, 0, 0};
    if (cell != NPOS) demorton(g.lv.code[cell], ijk);
    col_ijk[j][0] = ijk[0];
    col_ijk[j][1] = ijk[1];
    col_ijk[j][2] = ijk[2];
  }
  __syncthreads();
  // resident operand: the BN multipoles (zero columns past the end of the class)
  const int kc = g.K / 2;  // 16-byte chunks per column
  for (int ch = tid; ch < BN * kc; ch += PA_THREADS) {
    const int j = ch / kc, q = (ch % kc) * 2;
    const uint32_t cell = col_cell[j];
    const bool ok = cell != NPOS;
    cp16z(Ws + j * wpad + q, g.W + (ok ? size_t(cell) * g.ldE + q : 0), ok);
  }
  cp_commit();

  const double* A = g.A + cls * g.a_class_stride;
  const int KT = g.K / PA_BK;
  const int MTILES = g.rowsA / PA_BM;
  // M-split (coarse levels): this CTA streams M-tiles [mt0, mt1) of the operator
  const int per = (MTILES + g.msplit - 1) / g.msplit;
  const int mt0 = blockIdx.z * per, mt1 = min(MTILES, mt0 + per);
  if (mt0 >= mt1) return;
  const int TOTAL = (mt1 - mt0) * KT;
  // ring producer position (tile, k-slice), advanced without divisions
  int pmt = mt0, pkt = 0, pstage = 0;
  auto load_next = [&]() {
    double* as = As + pstage * PA_BM * PA_SPAD;
    const double* src = A + size_t(pmt * PA_BM) * g.lda + pkt * PA_BK;
    for (int ch = tid; ch < PA_BM * (PA_BK / 2); ch += PA_THREADS) {
      const int r = ch / (PA_BK / 2), q = (ch % (PA_BK / 2)) * 2;
      cp16(as + r * PA_SPAD + q, src + size_t(r) * g.lda + q);
    }
    if (++pkt == KT) { pkt = 0; ++pmt; }
    if (++pstage == PA_ST) pstage = 0;
  };
#pragma unroll
  for (int s = 0; s < PA_ST - 1; ++s) {
    if (s < TOTAL) load_next();
    cp_commit();
  }

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // epilogue tables of the current M-tile, fetched early so their latency hides
  // behind the tile's DMMAs: per row {destination column, vector index or -1}, and the
  // tile's vector slots feeding the (vector, column) -> target lookup
  const int kt_fill = KT / 2;
  int4 rowinfo[MT];  // consumed only by the tile's epilogue, KT k-slices after the load
  int slot_e0 = -1, slot_e1 = -1;
  int mt = mt0, kt = 0, stage = 0;
  for (int t = 0; t < TOTAL; ++t) {
    cp_wait<PA_ST - 2>();
    __syncthreads();
    if (t + PA_ST - 1 < TOTAL) load_next();
    cp_commit();
    uint32_t* tg = tgt;
    if (kt == 0) {
#pragma unroll
      for (int i = 0; i < MT; ++i) rowinfo[i] = __ldg(g.rowA + cls * g.rowsA + mt * PA_BM + wm * WTM + i * 8 + gq);
      const int* vec = g.tileVec + (size_t(cls) * MTILES + mt) * g.vtMax;
      slot_e0 = tid < g.vtMax * BN ? __ldg(vec + tid / BN) : -1;
      slot_e1 = tid + PA_THREADS < g.vtMax * BN ? __ldg(vec + (tid + PA_THREADS) / BN) : -1;
    }
    if (kt == kt_fill) {
      // one lookup per (vector, source column) of this M-tile: target = source - v.
      // (Looking the first two entries up before this slice's DMMAs and storing them after,
      // so the lookups' loads wait behind the DMMAs: 100 -> 118 registers, config-B M2L
      // 12.33 -> 12.40 ms, same fields bit for bit; tools/gpu/gpu_r02at.sh. Not adopted.)
      const int* vec = g.tileVec + (size_t(cls) * MTILES + mt) * g.vtMax;
      int u = 0;
      for (int e = tid; e < g.vtMax * BN; e += PA_THREADS, ++u) {
        const int j = e % BN;
        const int slot = u == 0 ? slot_e0 : u == 1 ? slot_e1 : __ldg(vec + e / BN);
        uint32_t tc = NPOS;
        if (slot >= 0 && col_cell[j] != NPOS)
          tc = find_ijk(g.lv, col_ijk[j][0] - (slot / 49 - 3), col_ijk[j][1] - ((slot / 7) % 7 - 3),
                        col_ijk[j][2] - (slot % 7 - 3));
        tg[e] = tc;
      }
      if (kt_fill == KT - 1) __syncthreads();
    }
    const double* as = As + stage * PA_BM * PA_SPAD + (wm * WTM + gq) * PA_SPAD + tq;
    const double* bs = Ws + (wn * WTN + gq) * wpad + kt * PA_BK + tq;
#pragma unroll
    for (int kk = 0; kk < PA_BK; kk += 4) {
      double a[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = as[i * 8 * PA_SPAD + kk];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = bs[j * 8 * wpad + kk];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    if (kt == KT - 1) {
      // scatter block v of source s to target s - v, target-side column info.x. The
      // targets of all the thread's elements are read first (one 8-byte LDS per column
      // pair), so the stores do not wait on a shared load each: the compiler cannot move
      // those loads above the global stores itself (generic pointers may alias)
      uint2 tcv[MT][NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const uint2* trow = reinterpret_cast<const uint2*>(tg + max(rowinfo[i].z, 0) * BN + wn * WTN + 2 * tq);
#pragma unroll
        for (int j = 0; j < NT; ++j) tcv[i][j] = rowinfo[i].x >= 0 ? trow[j * 4] : make_uint2(NPOS, NPOS);
      }
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        double* yrow = g.Yt + rowinfo[i].y;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          if (tcv[i][j].x != NPOS) yrow[size_t(tcv[i][j].x) * g.ldY] = acc[i][j][0];
          if (tcv[i][j].y != NPOS) yrow[size_t(tcv[i][j].y) * g.ldY] = acc[i][j][1];
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
      }
    }
    if (++stage == PA_ST) stage = 0;
    if (++kt == KT) { kt = 0; ++mt; }
  }
  cp_wait<0>();
}

// Phase A, streamed (phase B's GEMM structure with phase A's scatter epilogue): a BM x BN
// tile of Y = M1_p (rows) x W (source columns), BOTH operands streamed in BK-wide k-slices
// through a cp.async ring, so each operator slice feeds BN = 64 columns even at l = 7
// (the W-resident kernel holds 24 there). The epilogue resolves one target per (vector of
// the tile, column) from a table filled before the main loop.
template <int BM, int BN, int WM, int WN, int STAGES, int BK>
__global__ void __launch_bounds__(WM* WN * 32) k_m2l_phase_a2(const GemmArgs g) {
  constexpr int T = WM * WN * 32;
  constexpr int WTM = BM / WM, WTN = BN / WN;
  constexpr int MT = WTM / 8, NT = WTN / 8;
  constexpr int SPAD = BK + 4;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                      // [STAGES][BM][SPAD]
  double* Bs = smem + STAGES * BM * SPAD;  // [STAGES][BN][SPAD]
  uint32_t* tgt = reinterpret_cast<uint32_t*>(Bs + STAGES * BN * SPAD);  // [vtMax2][BN]
  __shared__ uint32_t col_cell[BN];

  const int cls = blockIdx.z;
  const uint32_t ncls = g.cls_off[cls + 1] - g.cls_off[cls];
  const uint32_t n0 = blockIdx.y * BN;
  if (n0 >= ncls) return;
  const int mt = blockIdx.x, m0 = mt * BM;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp / WN, wn = warp % WN;
  const int gq = lane >> 2, tq = lane & 3;

  for (int j = tid; j < BN; j += T) col_cell[j] = (n0 + j < ncls) ? g.cls_cells[g.cls_off[cls] + n0 + j] : NPOS;
  __syncthreads();

  const double* A = g.A + cls * g.a_class_stride + size_t(m0) * g.lda;
  const int KT = g.K / BK;
  auto load_tile = [&](int stage, int kt) {
    const int k0 = kt * BK;
    double* as = As + stage * BM * SPAD;
    double* bs = Bs + stage * BN * SPAD;
    for (int ch = tid; ch < BM * (BK / 2); ch += T) {
      const int r = ch / (BK / 2), q = (ch % (BK / 2)) * 2;
      cp16(as + r * SPAD + q, A + size_t(r) * g.lda + k0 + q);
    }
    for (int ch = tid; ch < BN * (BK / 2); ch += T) {
      const int j = ch / (BK / 2), q = (ch % (BK / 2)) * 2;
      const uint32_t cell = col_cell[j];
      const bool ok = cell != NPOS;
      cp16z(bs + j * SPAD + q, g.W + (ok ? size_t(cell) * g.ldE + k0 + q : 0), ok);
    }
  };
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < KT) load_tile(st, st);
    cp_commit();
  }
  // target of (vector of this tile, column): source - v, while the first slices load
  const int* vec = g.tileVec2 + (size_t(cls) * (g.rowsA / BM) + mt) * g.vtMax2;
  for (int e = tid; e < g.vtMax2 * BN; e += T) {
    const int j = e % BN, slot = __ldg(vec + e / BN);
    uint32_t tc = NPOS;
    const uint32_t cell = col_cell[j];
    if (slot >= 0 && cell != NPOS) {
      int ijk[3];
      demorton(g.lv.code[cell], ijk);
      tc = find_ijk(g.lv, ijk[0] - (slot / 49 - 3), ijk[1] - ((slot / 7) % 7 - 3), ijk[2] - (slot % 7 - 3));
    }
    tgt[e] = tc;
  }
  int4 rowinfo[MT];
#pragma unroll
  for (int i = 0; i < MT; ++i) rowinfo[i] = __ldg(g.rowA + cls * g.rowsA + m0 + wm * WTM + i * 8 + gq);

  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kt = 0; kt < KT; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int pf = kt + STAGES - 1;
    if (pf < KT) load_tile(pf % STAGES, pf);
    cp_commit();
    const double* as = As + (kt % STAGES) * BM * SPAD + (wm * WTM + gq) * SPAD + tq;
    const double* bs = Bs + (kt % STAGES) * BN * SPAD + (wn * WTN + gq) * SPAD + tq;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[MT], b[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) a[i] = as[i * 8 * SPAD + kk];
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = bs[j * 8 * SPAD + kk];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_wait<0>();
  // scatter block v of source s to target s - v (target-side column rowinfo.y)
#pragma unroll
  for (int i = 0; i < MT; ++i) {
    if (rowinfo[i].x < 0) continue;
    const uint32_t* trow = tgt + rowinfo[i].w * BN;
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t tcell = trow[wn * WTN + j * 8 + 2 * tq + e];
        if (tcell != NPOS) g.Yt[size_t(tcell) * g.ldY + rowinfo[i].y] = acc[i][j][e];
      }
  }
}

// Phase B tiles. Measured (evaluation ms at B / C, tools/gpu/gpu_r02ac.sh): 3-stage ring of
// 16-wide slices 24.81 / 81.20, 2-stage 16-wide 24.80 / 80.86, 128 x 128 tiles with 8 warps
// 25.04 / 81.24 (16-wide slices 25.25 / 82.44), against 24.60 / 80.28 for 128 x 64, 2-stage
// 32-wide slices.
constexpr int B_BM = 128, B_BN = 64, B_WM = 4, B_WN = 2, B_ST = 2, B_BK = 32;

}  // namespace

void m2l_free(fmmgpu_ctx* c) {
  auto& T = c->m2l;
  if (T.dM1) cudaFree(T.dM1);
  if (T.dM2) cudaFree(T.dM2);
  if (T.dRowA) cudaFree(T.dRowA);
  if (T.dTileVec) cudaFree(T.dTileVec);
  T.dTileVec = nullptr;
  if (T.dTileVec2) cudaFree(T.dTileVec2);
  T.dTileVec2 = nullptr;
  if (T.dKslot) cudaFree(T.dKslot);
  T.dM1 = T.dM2 = nullptr;
  T.dRowA = nullptr;
  T.dKslot = nullptr;
}

// Builds transport tables and the stacked per-parity operators from T.u/sigma/v.
void m2l_setup(fmmgpu_ctx* c, bool compute) {
  auto& T = c->m2l;
  const int l = c->order, n3 = c->l3;
  if (compute) compute_factors(c);
  // transport (m2l.cpp:146-163)
  std::fill(T.mult, T.mult + 16, 0);
  for (int s = 0; s < 343; ++s) {
    T.canonical[s] = -1;
    T.perm[s].clear();
    int v[3];
    slot_vec(s, v);
    if (std::max({std::abs(v[0]), std::abs(v[1]), std::abs(v[2])}) < 2) continue;
    int perm[3], sign[3];
    const int cl = canonicalize_host(v, perm, sign);
    T.canonical[s] = cl;
    T.perm[s] = grid_perm(perm, sign, l);
    ++T.mult[cl];
  }
  // target-side stacking per parity q: offB[q][slot]
  std::vector<int> offB(8 * 343, -1), offA(8 * 343, -1);
  int R = -1;
  for (int q = 0; q < 8; ++q) {
    int off = 0;
    for (int s = 0; s < 343; ++s) {
      int v[3];
      slot_vec(s, v);
      if (!admissible_for_target(v, q)) continue;
      offB[q * 343 + s] = off;
      off += T.rank[T.canonical[s]];
    }
    if (R < 0) R = off;
    if (off != R) throw Error(FMMGPU_LOGIC_ERROR, "M2L stack size differs across parity classes");
  }
  // source-side stacking per parity p: vectors with target s - v of parity p ^ par(v)
  for (int p = 0; p < 8; ++p) {
    int off = 0;
    for (int s = 0; s < 343; ++s) {
      int v[3];
      slot_vec(s, v);
      if (!admissible_for_target(v, p ^ vec_parity(v))) continue;
      offA[p * 343 + s] = off;
      off += T.rank[T.canonical[s]];
    }
    if (off != R) throw Error(FMMGPU_LOGIC_ERROR, "M2L source stack size mismatch");
  }
  T.R = R;
  T.ldY = round_up(R, 32);
  // 64-row M-tiles x 64 resident columns, 2-stage ring of 32-wide k-slices for l <= 5;
  // streamed 128 x 64 tiles (k_m2l_phase_a2) above. Earlier W-resident shapes at l = 7
  // (config C per evaluation, before the streamed kernel): 128 x 16 / 3 stages 96.9 ms,
  // 64 x 32 / 2 stages 95.8 (16 x 16 warp tiles) or 95.1 (32 x 8), 128 x 24 / 2 stages
  // 94.0. Config B with 128 x 64 / 2 stages (32 x 32 warp tiles): 27.90 vs
  // 27.78 ms per evaluation. Measured at the config-B leaf (phase A + B): 128 x 64 / 2 stages 15.9 ms,
  // 128 x 32 / 3 stages 12.6 ms, vs 11.9 ms for 64 x 64 / 4 stages.
  T.bmA = c->ldE <= 128 ? 64 : 128;
  T.rowsA = round_up(R, 128);  // whole 64- and 128-row tiles (2432 at l = 5, as round_up(R, 64))
  T.rowsB = round_up(n3, B_BM);
  std::vector<double> M1(size_t(8) * T.rowsA * c->ldE, 0.0), M2(size_t(8) * T.rowsB * T.ldY, 0.0);
  std::vector<int4> rowA(size_t(8) * T.rowsA, make_int4(-1, 0, 0, 0));
  std::vector<int> kslot(size_t(8) * T.ldY, -1);
  for (int p = 0; p < 8; ++p)
    for (int s = 0; s < 343; ++s) {
      const int oa = offA[p * 343 + s];
      if (oa >= 0) {
        int v[3];
        slot_vec(s, v);
        const int cl = T.canonical[s], r = T.rank[cl];
        const int q = p ^ vec_parity(v);
        const int ob = offB[q * 343 + s];
        for (int k = 0; k < r; ++k) {
          double* row = &M1[(size_t(p) * T.rowsA + oa + k) * c->ldE];
          for (int n = 0; n < n3; ++n) row[n] = T.sigma[cl][k] * T.v[cl][size_t(T.perm[s][n]) * r + k];
          rowA[size_t(p) * T.rowsA + oa + k] = make_int4(s, ob + k, 0, 0);
        }
      }
      const int ob = offB[p * 343 + s];  // here p plays the target parity q
      if (ob >= 0) {
        const int cl = T.canonical[s], r = T.rank[cl];
        for (int k = 0; k < r; ++k) {
          kslot[size_t(p) * T.ldY + ob + k] = s;
          for (int m = 0; m < n3; ++m)
            M2[(size_t(p) * T.rowsB + m) * T.ldY + ob + k] = T.u[cl][size_t(T.perm[s][m]) * r + k];
        }
      }
    }
  m2l_free(c);
  fmmgpu_invalidate_graph(c);
  for (auto& L : c->lv)  // the Yt layout depends on the ranks: drop stale intermediates
    if (L.yt) {
      FMM_CUDA(cudaFree(L.yt));
      L.yt = nullptr;
    }
  for (auto& p : c->yt_keep)
    if (p) {
      FMM_CUDA(cudaFree(p));
      p = nullptr;
    }
  FMM_CUDA(cudaMalloc(&T.dM1, M1.size() * sizeof(double)));
  FMM_CUDA(cudaMalloc(&T.dM2, M2.size() * sizeof(double)));
  // per 64-row M-tile of phase A: the distinct vectors it holds (rows of one vector
  // are consecutive), so the epilogue resolves one target per (vector, column)
  const int PA_BM = T.bmA;
  const int mtiles = T.rowsA / PA_BM;
  T.vtMax = 1;
  std::vector<std::vector<int>> tv(size_t(8) * mtiles);
  for (int p = 0; p < 8; ++p)
    for (int mt = 0; mt < mtiles; ++mt) {
      auto& list = tv[size_t(p) * mtiles + mt];
      for (int r = 0; r < PA_BM; ++r) {
        int4& e = rowA[size_t(p) * T.rowsA + mt * PA_BM + r];
        if (e.x < 0) continue;
        if (list.empty() || list.back() != e.x) list.push_back(e.x);
        e.z = static_cast<int>(list.size()) - 1;
      }
      T.vtMax = std::max<int>(T.vtMax, static_cast<int>(list.size()));
    }
  {  // 128-row tiles of the streamed phase A: vector index in rowA.w
    const int mt2 = T.rowsA / 128;
    T.vtMax2 = 1;
    std::vector<std::vector<int>> tv2(size_t(8) * mt2);
    for (int p = 0; p < 8; ++p)
      for (int mt = 0; mt < mt2; ++mt) {
        auto& list = tv2[size_t(p) * mt2 + mt];
        for (int r = 0; r < 128; ++r) {
          int4& e = rowA[size_t(p) * T.rowsA + mt * 128 + r];
          if (e.x < 0) continue;
          if (list.empty() || list.back() != e.x) list.push_back(e.x);
          e.w = static_cast<int>(list.size()) - 1;
        }
        T.vtMax2 = std::max<int>(T.vtMax2, static_cast<int>(list.size()));
      }
    std::vector<int> tileVec2(size_t(8) * mt2 * T.vtMax2, -1);
    for (size_t i = 0; i < tv2.size(); ++i) std::copy(tv2[i].begin(), tv2[i].end(), tileVec2.begin() + i * T.vtMax2);
    FMM_CUDA(cudaMalloc(&T.dTileVec2, tileVec2.size() * sizeof(int)));
    FMM_CUDA(cudaMemcpy(T.dTileVec2, tileVec2.data(), tileVec2.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  std::vector<int> tileVec(size_t(8) * mtiles * T.vtMax, -1);
  for (size_t i = 0; i < tv.size(); ++i)
    std::copy(tv[i].begin(), tv[i].end(), tileVec.begin() + i * T.vtMax);
  FMM_CUDA(cudaMalloc(&T.dTileVec, tileVec.size() * sizeof(int)));
  FMM_CUDA(cudaMemcpy(T.dTileVec, tileVec.data(), tileVec.size() * sizeof(int), cudaMemcpyHostToDevice));
  FMM_CUDA(cudaMalloc(&T.dRowA, rowA.size() * sizeof(int4)));
  FMM_CUDA(cudaMalloc(&T.dKslot, kslot.size() * sizeof(int)));
  FMM_CUDA(cudaMemcpy(T.dM1, M1.data(), M1.size() * sizeof(double), cudaMemcpyHostToDevice));
  FMM_CUDA(cudaMemcpy(T.dM2, M2.data(), M2.size() * sizeof(double), cudaMemcpyHostToDevice));
  FMM_CUDA(cudaMemcpy(T.dRowA, rowA.data(), rowA.size() * sizeof(int4), cudaMemcpyHostToDevice));
  FMM_CUDA(cudaMemcpy(T.dKslot, kslot.data(), kslot.size() * sizeof(int), cudaMemcpyHostToDevice));
  std::vector<int> canon(T.canonical, T.canonical + 343);
  if (!c->d_canon) FMM_CUDA(cudaMalloc(&c->d_canon, 343 * sizeof(int)));
  FMM_CUDA(cudaMemcpy(c->d_canon, canon.data(), 343 * sizeof(int), cudaMemcpyHostToDevice));
  (void)l;
}

void launch_m2l(fmmgpu_ctx* c, int v, cudaStream_t s) {
  auto& T = c->m2l;
  const Level& L = c->lv[v];
  if (L.n == 0) return;
  Level& Lm = c->lv[v];
  if (!Lm.yt && L.full && v < 22 && c->yt_keep[v] && c->yt_keep_n[v] == L.n) {
    Lm.yt = c->yt_keep[v];  // same full level as a previous tree: absent-source blocks still zero
    c->yt_keep[v] = nullptr;
  }
  if (!Lm.yt) {  // per-level compressed intermediates; zero = "no source" (see phase B)
    FMM_CUDA(cudaMallocAsync(&Lm.yt, size_t(L.n) * T.ldY * sizeof(double), s));
    FMM_CUDA(cudaMemsetAsync(Lm.yt, 0, size_t(L.n) * T.ldY * sizeof(double), s));
  }
  GemmArgs g{};
  g.lv = L.view(v);
  // phase A runs over the sources (partitioned: those with an owned target), phase B
  // over the targets (partitioned: the owned ones)
  g.cls_cells = L.srcA ? L.srcA : L.cls_cells;
  std::copy(L.srcA ? L.srcA_off : L.cls_off, (L.srcA ? L.srcA_off : L.cls_off) + 9, g.cls_off);
  g.W = L.multipole;
  g.ldE = c->ldE;
  g.Yt = Lm.yt;
  g.ldY = T.ldY;
  g.rowA = T.dRowA;
  g.tileVec = T.dTileVec;
  g.vtMax = T.vtMax;
  g.tileVec2 = T.dTileVec2;
  g.vtMax2 = T.vtMax2;
  g.rowsA = T.rowsA;
  g.kslot = T.dKslot;
  g.local = L.local_own;
  g.ow = c->ow ? 1 : 0;
  g.l3 = c->l3;
  g.scale = 1.0 / (c->root[3] / static_cast<double>(uint64_t{1} << v));  // bench.cpp:233-234
  uint32_t maxcls = 0;
  for (int q = 0; q < 8; ++q) maxcls = std::max(maxcls, g.cls_off[q + 1] - g.cls_off[q]);
  if (maxcls) {
    g.A = T.dM1;
    g.lda = c->ldE;
    g.a_class_stride = size_t(T.rowsA) * c->ldE;
    g.K = c->ldE;
    // BN chosen so the resident multipoles + the A ring fit two CTAs per SM
    auto launch = [&](auto kern, int bn, int PA_BM, int PA_ST, int bk = 16, int threads = 256) {
      const size_t smem = sizeof(double) * (size_t(bn) * (g.K + 4) + size_t(PA_ST) * PA_BM * (bk + 4)) +
                          sizeof(uint32_t) * size_t(T.vtMax) * bn;
      FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      // M-split so coarse levels still put >= 2 CTAs on every SM
      const uint32_t ncols = 8u * ((maxcls + bn - 1) / bn);
      const int mtiles = T.rowsA / PA_BM;
      int ms = 1;
      static const uint32_t waves = [] {  // FMMGPU_M2L_WAVES: minimum CTA waves (2 per SM) before M-splitting stops
        const char* e = std::getenv("FMMGPU_M2L_WAVES");
        return e ? static_cast<uint32_t>(std::atoi(e)) : 2u;  // config B: 28.55 vs 28.76 ms (1 wave)
      }();
      while (ms < mtiles && ncols * ms < waves * 2u * 148u) ++ms;
      // (forcing an M-split of 2 / 4 / 8 on full levels so fewer classes' operators are live
      // in L2 at once: config C 88.66 / 88.26 / 88.31 vs 88.81 ms, config B 24.60 / 24.75 vs
      // 24.56 -- not adopted)
      g.msplit = ms;
      static const int cls_fast = [] {  // FMMGPU_M2L_CLS_FAST=0: class-slowest order (A/B aid)
        const char* e = std::getenv("FMMGPU_M2L_CLS_FAST");
        return e ? std::atoi(e) : 1;
      }();
      g.cls_fast = cls_fast;
      dim3 grid = cls_fast ? dim3(8, (maxcls + bn - 1) / bn, ms) : dim3((maxcls + bn - 1) / bn, 8, ms);
      kern<<<grid, threads, smem, s>>>(g);
      FMM_CUDA(cudaGetLastError());
    };
    // l <= 5: 32-wide k-slices through a 2-stage ring (config B: 27.26 vs 27.81 ms per
    // evaluation with 16-wide slices and 4 stages; a 3-stage 32-wide ring no longer fits
    // two CTAs per SM)
    // Also measured (tools/gpu/gpu_r02o.sh, evaluation ms at config B / C): 64 x 64 with 4
    // warps of 32 x 32 (24.84 vs 24.53), 64 x 32 with 4 warps and 3 CTAs per SM (24.62), the
    // same with a 3-stage ring (25.79); at l = 7, 128 x 32 with one CTA per SM (97.76 vs 88.76).
    // Round 2: 128-row M-tiles with 8 warps of 32 x 32 and a 2-stage ring of 16-wide slices
    // (two CTAs per SM, 128 registers; tools/gpu/gpu_r02au.sh): M2L 12.85 vs 12.33 ms at B.
    // l >= 6: the streamed kernel (config C 87.94 -> 80.21 ms per evaluation, l = 6
    // 49.06 -> 45.42; at l = 5 it measured slower, 25.30 vs 24.59 ms at B). Streamed
    // shapes also measured at C: 128 x 128 with 16 warps (84.42), 3-stage ring (88.50),
    // 128 x 128 with 8 warps and 16-wide slices (86.04).
    auto launch2 = [&](auto kern, int st, int bk, int bn, int threads) {
      const size_t smem = sizeof(double) * size_t(st) * (128 + bn) * (bk + 4) + sizeof(uint32_t) * T.vtMax2 * bn;
      FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      dim3 grid(T.rowsA / 128, (maxcls + bn - 1) / bn, 8);
      kern<<<grid, threads, smem, s>>>(g);
      FMM_CUDA(cudaGetLastError());
    };
    if (T.bmA == 64) launch(k_m2l_phase_a<64, 2, 64, 2, 4, 32>, 64, 64, 2, 32);
    else launch2(k_m2l_phase_a2<128, 64, 4, 2, 2, 32>, 2, 32, 64, 256);
  }
  g.cls_cells = L.tgtB ? L.tgtB : L.cls_cells;
  std::copy(L.tgtB ? L.tgtB_off : L.cls_off, (L.tgtB ? L.tgtB_off : L.cls_off) + 9, g.cls_off);
  maxcls = 0;
  for (int q = 0; q < 8; ++q) maxcls = std::max(maxcls, g.cls_off[q + 1] - g.cls_off[q]);
  if (maxcls) {
    g.A = T.dM2;
    g.lda = T.ldY;
    g.a_class_stride = size_t(T.rowsB) * T.ldY;
    g.K = T.ldY;
    g.ncells = L.n;
    // deterministic split-K when the level has too few column tiles to fill 2 CTAs/SM
    const int mtiles = T.rowsB / B_BM;
    const uint32_t ctas = 8u * ((maxcls + B_BN - 1) / B_BN) * mtiles;
    const int kt = T.ldY / B_BK;
    int ks = 1;
    static const uint32_t waves = [] {
      const char* e = std::getenv("FMMGPU_M2L_WAVES");
      return e ? static_cast<uint32_t>(std::atoi(e)) : 2u;  // config B: 28.55 vs 28.76 ms (1 wave)
    }();
    while (ks < 16 && ctas * ks < waves * 2u * 148u && kt / (2 * ks) >= 8) ks *= 2;
    g.ksplit = ks;
    const int sb = v == c->height - 1 ? 1 : 0;  // the leaf may run beside the coarse levels
    if (ks > 1) {  // own buffer (not the shared scratch): captured graphs keep this pointer
      const size_t bytes = sizeof(double) * ks * size_t(L.n) * c->ldE;
      if (bytes > c->splitk_cap[sb]) {
        if (c->capturing) throw Error(FMMGPU_LOGIC_ERROR, "split-K buffer growth during graph capture");
        if (c->d_splitk[sb]) FMM_CUDA(cudaFreeAsync(c->d_splitk[sb], s));
        FMM_CUDA(cudaMallocAsync(&c->d_splitk[sb], bytes, s));
        c->splitk_cap[sb] = bytes;
        fmmgpu_invalidate_graph(c);
      }
    }
    g.part = ks > 1 ? c->d_splitk[sb] : nullptr;
    // M-tiles of 128 rows; the rows past the last whole tile go to a 96- or 64-row tail
    // tile when that covers them (l = 7: 343 rows as 2 x 128 + 96 = 352 instead of 384, 11%
    // fewer DMMAs; l = 6: 128 + 96 = 224 instead of 256)
    auto run = [&](auto kern, int bm, int threads, int tiles, int row0) {
      if (tiles <= 0) return;
      const size_t smem = sizeof(double) * B_ST * (bm + B_BN) * (B_BK + 4);
      FMM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      g.rowB0 = row0;
      dim3 grid(tiles, (maxcls + B_BN - 1) / B_BN, 8 * ks);
      kern<<<grid, threads, smem, s>>>(g);
      FMM_CUDA(cudaGetLastError());
    };
    const int full = c->l3 / B_BM, tail = c->l3 - full * B_BM;
    const int whole = tail > 96 ? full + 1 : full;
    run(k_m2l_phase_b<B_BM, B_BN, B_WM, B_WN, B_ST, B_BK>, B_BM, B_WM * B_WN * 32, whole, 0);
    if (tail > 0 && tail <= 64) {
      run(k_m2l_phase_b<64, B_BN, 2, B_WN, B_ST, B_BK>, 64, 2 * B_WN * 32, 1, full * B_BM);
      if (full) ++c->launches;
    } else if (tail > 64 && tail <= 96) {
      run(k_m2l_phase_b<96, B_BN, 3, B_WN, B_ST, B_BK>, 96, 3 * B_WN * 32, 1, full * B_BM);
      if (full) ++c->launches;
    }
    if (ks > 1) {
      const uint32_t ntg = g.cls_off[8];
      const uint64_t tot = uint64_t(ntg) * c->ldE;
      k_m2l_splitk_reduce<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, s>>>(
          g.part, ks, L.n, c->ldE, c->l3, g.scale, g.cls_cells, ntg, L.local_own, c->ow ? 1 : 0);
      FMM_CUDA(cudaGetLastError());
      ++c->launches;
    }
  }
  c->launches += 2;
}

}  // namespace fmmgpu

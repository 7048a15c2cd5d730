// Assembled sum factorization for p = 3, q = 4 (the headline configs C3/C5) on
// FP64 tensor cores: every contraction is a DMMA.8x8x4 GEMM whose K = 4 is
// exactly one element's quadrature points, and the inter-element (assembly)
// sum is done in the accumulator registers.
//
// Same mathematics and tiling as k_gsf3 (iga_gsf.cu header): one CTA per
// TA x TB = 2 x 4 row pencils, streaming the elements e2 of the fastest axis.
//
// Per element along an axis, the element-local product  C[x][(r,s)] =
// sum_k A[x][k] T(r,k) T(s,k)  has its (r,s) pairs on the MMA N axis.  The
// 16 pairs of p = 3 fit two 8-column n-tiles so that the quad lane t holds the
// four columns (r, s = (r+t) mod 4), r = 0..3: one column per r.  The global
// row offset of column (r,s) is then a compile-time function of (element, r)
// and its band offset d = s - r + 3 takes one of two lane-constant values
// (d = 3+t if r < 4-t, else t-1), so each lane accumulates its contributions
// to the assembled values in two registers per destination row -- no shared
// memory read-modify-write, no atomics, and the assembly is exact-order
// deterministic.
//
//   stage A (axis 0): C[(g1,k2)][(r,s)] = sum_k0 W[la,k0][(g1,k2)] PA_la[k0][(r,s)]
//                     -> X_T[ia = la+r-3][d0][(g1,k2)]                (T = V, D)
//   stage B (axis 1): C[(a0,k2)][(r,s)] = sum_k1 X_T[a0][(lb,k1,k2)] PB_lb[k1][(r,s)]
//                     -> Y_A/Y_B[(a0, ib = lb+r-3, d1)][k2]
//   stage S (axis 2): C[c][(r,s)] = sum_k2 Y[c][k2] Z_e2[k2][(r,s)]
//                     -> R[c][row e2+r][d2]  (registers, rolling over 4 rows)
#include "iga_args.cuh"
#include "iga_dispatch.cuh"

namespace iga {
namespace p3 {

constexpr int P = 3, M = 4, Q = 4, NB = 7;
constexpr int TA = 2, TB = 4;
constexpr int LA = TA + P, LB = TB + P;  // element windows (5, 7)
constexpr int GB = LB * Q;               // axis-1 quadrature points in the window (28)
constexpr int NCOL = GB * Q;             // (g1, k2) columns (112)
constexpr int WP = NCOL + 4;             // W row pitch (== 4 mod 16: conflict-free A loads)
constexpr int NA0 = TA * NB;             // (ia, d0) rows (14)
constexpr int NCOMBO = NA0 * TB * NB;    // (ia, d0, ib, d1) combos (392)
constexpr int YP = NCOMBO + 4;           // Y pitch (== 12 mod 16: conflict-free A loads)
constexpr int NT = 512;                  // threads (16 warps)
constexpr int NW = NT / 32;
constexpr int MT_A = NCOL / 8;           // 14 m-tiles of (g1,k2) columns
constexpr int MT_B = NA0 * Q / 8;        // 7 m-tiles of (a0,k2) rows
constexpr int MT_S = NCOMBO / 8;         // 49 m-tiles of combos
constexpr int MT_S_PER_WARP = (MT_S + NW - 1) / NW;  // 4
constexpr int NPEN = TA * TB;            // row pencils (I0, I1) of the tile

// shared memory layout (doubles)
constexpr int OFF_W = 0;                          // [LA*Q][WP]
constexpr int OFF_X = OFF_W + LA * Q * WP;        // [2 types][NA0][NCOL]
constexpr int OFF_Y = OFF_X + 2 * NA0 * NCOL;     // [2 accs * Q][YP]
constexpr int OFF_BA = OFF_Y + 2 * Q * YP;        // [2 types][LA][2 nt][32]
constexpr int OFF_BB = OFF_BA + 2 * LA * 2 * 32;  // [2 prods][LB][2 nt][32]
constexpr int OFF_WQ = OFF_BB + 2 * LB * 2 * 32;  // weights [Q]
constexpr int OFF_PB = OFF_WQ + Q;                // pencil row-pointer bases (int64) [NPEN]
constexpr int OFF_PC = OFF_PB + NPEN;             // pencil c0*c1 (as double-sized slots) [NPEN]
constexpr int SMEM_DOUBLES = OFF_PC + NPEN;
constexpr size_t SMEM_BYTES = SMEM_DOUBLES * sizeof(double);

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0,
                                     double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Is any column k in {2nt, 2nt+1} of window element l mapped to a destination
// index l + k - P inside [lo, hi)?
__host__ __device__ constexpr bool nt_useful(int l, int nt, int lo, int hi) {
  return (l + 2 * nt - P >= lo && l + 2 * nt - P < hi) ||
         (l + 2 * nt + 1 - P >= lo && l + 2 * nt + 1 - P < hi);
}

// B-fragment column mapping: lane (g, t) holds B[k=t][n=g]; column n of n-tile nt
// is the pair (r, s) = (2nt + (n&1), (r + (n>>1)) & 3).
__device__ __forceinline__ int bcol_r(int nt, int g) { return 2 * nt + (g & 1); }
__device__ __forceinline__ int bcol_s(int nt, int g) { return (bcol_r(nt, g) + (g >> 1)) & 3; }

struct Ctx {
  double* W;
  double* X;
  double* Y;
  const double* BA;
  const double* BB;
  int lane, warp, g, t;
  bool stiff, smass;
};

// Clamp helper for compile-time-resolved accumulator references.
__host__ __device__ constexpr int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ---- stage A unit: m-tile mt of (g1,k2) columns, type ty (0 = values, 1 = derivatives).
// Per-column accumulators acc[ia][k] are the DMMA C operands (in-place assembly over la).
__device__ __forceinline__ void stage_a_unit(const Ctx& c, int mt, int ty) {
  double acc[TA][4];
#pragma unroll
  for (int ia = 0; ia < TA; ++ia)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[ia][k] = 0.0;
#pragma unroll
  for (int la = 0; la < LA; ++la) {
    const double av = c.W[(la * Q + c.t) * WP + mt * 8 + c.g];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      if (!nt_useful(la, nt, 0, TA)) continue;
      const int ia0 = la + 2 * nt - P, ia1 = ia0 + 1;
      double z0 = 0.0, z1 = 0.0;
      double& r0 = (ia0 >= 0 && ia0 < TA) ? acc[clampi(ia0, 0, TA - 1)][2 * nt] : z0;
      double& r1 = (ia1 >= 0 && ia1 < TA) ? acc[clampi(ia1, 0, TA - 1)][2 * nt + 1] : z1;
      dmma(r0, r1, av, c.BA[((ty * LA + la) * 2 + nt) * 32 + c.lane], r0, r1);
    }
  }
  const int col = mt * 8 + c.g, t = c.t;
#pragma unroll
  for (int ia = 0; ia < TA; ++ia) {
    double hi = 0.0, lo = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < 4 - t) hi += acc[ia][k]; else lo += acc[ia][k];
    }
    c.X[(ty * NA0 + ia * NB + P + t) * NCOL + col] = hi;
    if (t > 0) c.X[(ty * NA0 + ia * NB + t - 1) * NCOL + col] = lo;
  }
}

// ---- stage B unit: m-tile mt of (a0,k2) rows, destination ib in {2H, 2H+1};
// per-column accumulators are the DMMA C operands (in-place assembly over lb).
template <int H>
__device__ __forceinline__ void stage_b_unit(const Ctx& c, int mt) {
  const int row = mt * 8 + c.g, a0 = row >> 2, k2 = row & 3, t = c.t;
  double yA[2][4], yB[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) yA[i][k] = yB[i][k] = 0.0;
#pragma unroll
  for (int lb = 2 * H; lb <= 2 * H + 4; ++lb) {
    const int xo = (lb * Q + t) * Q + k2;
    const double xv = c.X[(0 * NA0 + a0) * NCOL + xo];
    const double xd = c.stiff ? c.X[(1 * NA0 + a0) * NCOL + xo] : 0.0;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      if (!nt_useful(lb, nt, 2 * H, 2 * H + 2)) continue;
      const int i0 = lb + 2 * nt - P - 2 * H, i1 = i0 + 1;
      const bool v0 = i0 >= 0 && i0 < 2, v1 = i1 >= 0 && i1 < 2;
      double z0 = 0.0, z1 = 0.0, z2 = 0.0, z3 = 0.0;
      double& a0r = v0 ? yA[clampi(i0, 0, 1)][2 * nt] : z0;
      double& a1r = v1 ? yA[clampi(i1, 0, 1)][2 * nt + 1] : z1;
      double& b0r = v0 ? yB[clampi(i0, 0, 1)][2 * nt] : z2;
      double& b1r = v1 ? yB[clampi(i1, 0, 1)][2 * nt + 1] : z3;
      const double vv = c.BB[((0 * LB + lb) * 2 + nt) * 32 + c.lane];
      if (c.stiff) {
        const double dd = c.BB[((1 * LB + lb) * 2 + nt) * 32 + c.lane];
        dmma(a0r, a1r, xd, vv, a0r, a1r);
        dmma(b0r, b1r, xv, vv, b0r, b1r);
        dmma(a0r, a1r, xv, dd, a0r, a1r);
      } else {
        dmma(a0r, a1r, xv, vv, a0r, a1r);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    double ah = 0.0, al = 0.0, bh = 0.0, bl = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < 4 - t) { ah += yA[i][k]; bh += yB[i][k]; }
      else { al += yA[i][k]; bl += yB[i][k]; }
    }
    const int ib = 2 * H + i;
    const int ch = (a0 * TB + ib) * NB + P + t;
    c.Y[(0 * Q + k2) * YP + ch] = ah;
    if (c.stiff) c.Y[(1 * Q + k2) * YP + ch] = bh;
    if (t > 0) {
      const int cl = (a0 * TB + ib) * NB + t - 1;
      c.Y[(0 * Q + k2) * YP + cl] = al;
      if (c.stiff) c.Y[(1 * Q + k2) * YP + cl] = bl;
    }
  }
}

// ---- stage S: element e2 along axis 2 into the rolling row accumulators
template <int PHI>
__device__ __forceinline__ void stage_s(const Ctx& c, double (&R)[MT_S_PER_WARP][4][2],
                                        const GsfArgs& a, int e2) {
  const int g = c.g, t = c.t;
  const double* V2 = a.V + (int64_t)e2 * M * Q;
  double b0[2], b1[2];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int r = bcol_r(nt, g), s = bcol_s(nt, g);
    b0[nt] = __ldg(V2 + r * Q + t) * __ldg(V2 + s * Q + t);
    b1[nt] = 0.0;
    if (c.stiff) {
      const double* D2 = a.D + (int64_t)e2 * M * Q;
      double z = __ldg(D2 + r * Q + t) * __ldg(D2 + s * Q + t);
      if (c.smass) z += b0[nt];
      b1[nt] = z;
    }
  }
#pragma unroll
  for (int i = 0; i < MT_S_PER_WARP; ++i) {
    const int mt = c.warp + i * NW;
    if (mt < MT_S) {
      const double a0 = c.Y[(0 * Q + t) * YP + mt * 8 + g];
      const double a1 = c.stiff ? c.Y[(1 * Q + t) * YP + mt * 8 + g] : 0.0;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        double c0, c1;
        dmma(c0, c1, a0, b0[nt], 0.0, 0.0);
        if (c.stiff) dmma(c0, c1, a1, b1[nt], c0, c1);
        // column k = 2nt + j has r = k: destination row e2 + k -> slot (PHI + k) & 3
        const int k0 = 2 * nt, k1 = 2 * nt + 1;
        if (k0 < 4 - t) R[i][(PHI + k0) & 3][0] += c0; else R[i][(PHI + k0) & 3][1] += c0;
        if (k1 < 4 - t) R[i][(PHI + k1) & 3][0] += c1; else R[i][(PHI + k1) & 3][1] += c1;
      }
    }
  }
}

// Row I2 (slot SL) is complete: each lane stores its (up to) two values per m-tile
// straight to the CSR row (neighbouring lanes cover contiguous row segments).
template <int SL>
__device__ __forceinline__ void flush(const Ctx& c, double (&R)[MT_S_PER_WARP][4][2],
                                      const int (&meta)[MT_S_PER_WARP], const int64_t* pb,
                                      const int* pc, const GsfArgs& a, int I2, int64_t N) {
  const int t = c.t;
  const int lod2 = max(0, P - I2);
  const int c2 = (int)band_cnt(I2, P, N);
  const int64_t pre2 = band_prefix(I2, P, N);
  const int dh = P + t - lod2, dl = t - 1 - lod2;
#pragma unroll
  for (int i = 0; i < MT_S_PER_WARP; ++i) {
    const int m = meta[i];
    if (m >= 0) {
      const int rc = m >> 16, b01 = m & 0xffff;
      double* row = a.values + pb[rc] + (int64_t)pc[rc] * pre2 + b01 * c2;
      if (dh >= 0 && dh < c2) row[dh] = R[i][SL][0];
      if (t > 0 && dl >= 0 && dl < c2) row[dl] = R[i][SL][1];
    }
    R[i][SL][0] = 0.0;
    R[i][SL][1] = 0.0;
  }
}

__device__ __forceinline__ void flush_any(int sl, const Ctx& c, double (&R)[MT_S_PER_WARP][4][2],
                                          const int (&meta)[MT_S_PER_WARP], const int64_t* pb,
                                          const int* pc, const GsfArgs& a, int I2, int64_t N) {
  switch (sl) {
    case 0: flush<0>(c, R, meta, pb, pc, a, I2, N); break;
    case 1: flush<1>(c, R, meta, pb, pc, a, I2, N); break;
    case 2: flush<2>(c, R, meta, pb, pc, a, I2, N); break;
    default: flush<3>(c, R, meta, pb, pc, a, I2, N); break;
  }
}

__device__ __forceinline__ void form_w(double* W, const double* wq, const GsfArgs& a, int e2,
                                       int i00, int i10, int e0lo, int e0hi, int tid) {
  const int K = a.K;
  for (int u = tid; u < LA * Q * NCOL; u += NT) {
    const int row = u / NCOL, col = u - row * NCOL;
    const int la = row >> 2, k0 = row & 3;
    const int g1 = col >> 2, k2 = col & 3, lb = g1 >> 2, k1 = g1 & 3;
    const int e0 = i00 - P + la, e1 = i10 - P + lb;
    double w = 0.0;
    if (e0 >= e0lo && e0 < e0hi && e1 >= 0 && e1 < K) {
      const double cf = a.coef ? __ldg(a.coef + (((int64_t)e0 * K + e1) * K + e2) * (Q * Q * Q) +
                                       (k0 * Q + k1) * Q + k2)
                               : a.coef_scalar;
      w = wq[k0] * wq[k1] * wq[k2] * a.jac * cf;
    }
    W[row * WP + col] = w;
  }
}

__global__ void __launch_bounds__(NT, 1) k_gsf3_p3(GsfArgs a) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  Ctx c;
  c.lane = tid & 31; c.warp = tid >> 5; c.g = c.lane >> 2; c.t = c.lane & 3;
  c.stiff = a.op != IGA_OP_MASS;
  c.smass = a.op == IGA_OP_STIFFNESS_MASS;
  c.W = sm + OFF_W; c.X = sm + OFF_X; c.Y = sm + OFF_Y; c.BA = sm + OFF_BA; c.BB = sm + OFF_BB;
  double* wq = sm + OFF_WQ;
  int64_t* pb = reinterpret_cast<int64_t*>(sm + OFF_PB);
  int* pc = reinterpret_cast<int*>(sm + OFF_PC);
  const int K = a.K;
  const int64_t N = (int64_t)K + P;
  const int tile0 = blockIdx.x / a.tiles1, tile1 = blockIdx.x % a.tiles1;
  const int i00 = a.plane_begin + tile0 * TA, i10 = tile1 * TB;
  const int e0lo = max(a.el_begin, 0), e0hi = min(a.el_end, K);

  // ---- constant B fragments of axes 0 and 1 (pair products of the window elements)
  double* BA = sm + OFF_BA;
  double* BB = sm + OFF_BB;
  for (int u = tid; u < 2 * LA * 2 * 32; u += NT) {
    const int ln = u & 31, nt = (u >> 5) & 1, la = (u >> 6) % LA, type = u / (64 * LA);
    const int gg = ln >> 2, tt = ln & 3, e0 = i00 - P + la;
    double v = 0.0;
    if (e0 >= 0 && e0 < K && (type == 0 || c.stiff)) {
      const double* T = (type == 0 ? a.V : a.D) + (int64_t)e0 * M * Q;
      v = T[bcol_r(nt, gg) * Q + tt] * T[bcol_s(nt, gg) * Q + tt];
    }
    BA[u] = v;
  }
  for (int u = tid; u < 2 * LB * 2 * 32; u += NT) {
    const int ln = u & 31, nt = (u >> 5) & 1, lb = (u >> 6) % LB, prod = u / (64 * LB);
    const int gg = ln >> 2, tt = ln & 3, e1 = i10 - P + lb;
    double v = 0.0;
    if (e1 >= 0 && e1 < K && (prod == 0 || c.stiff)) {
      const double* T = (prod == 0 ? a.V : a.D) + (int64_t)e1 * M * Q;
      v = T[bcol_r(nt, gg) * Q + tt] * T[bcol_s(nt, gg) * Q + tt];
    }
    BB[u] = v;
  }
  if (tid < Q) wq[tid] = a.weights[tid];
  if (tid < NPEN) {
    const int64_t I0 = i00 + tid / TB, I1 = i10 + tid % TB;
    // rowptr of (I0, I1, 0) relative to the launch's first row; c0*c1 per I2-prefix unit
    pb[tid] = (I0 < N && I1 < N) ? rowptr3(I0, I1, 0, P, N) - a.base : 0;
    pc[tid] = (I0 < N && I1 < N) ? (int)(band_cnt(I0, P, N) * band_cnt(I1, P, N)) : 0;
  }

  // per-lane flush metadata of its stage-S m-tiles: staging pencil rc and the (d0,d1)
  // block offset b01 = (d0-lo0)*c1 + (d1-lo1) in the CSR row; -1 if the combo is outside
  int meta[MT_S_PER_WARP];
#pragma unroll
  for (int i = 0; i < MT_S_PER_WARP; ++i) {
    const int mt = c.warp + i * NW;
    meta[i] = -1;
    if (mt < MT_S) {
      const int cb = mt * 8 + c.g;
      const int d1 = cb % NB, ib = (cb / NB) % TB, a0 = cb / (NB * TB);
      const int d0 = a0 % NB, ia = a0 / NB;
      const int I0 = i00 + ia, I1 = i10 + ib;
      if (I0 < a.plane_end && I1 < N) {
        const int lod0 = max(0, P - I0), lod1 = max(0, P - I1);
        const int c0 = (int)band_cnt(I0, P, N), c1 = (int)band_cnt(I1, P, N);
        if (d0 >= lod0 && d0 < lod0 + c0 && d1 >= lod1 && d1 < lod1 + c1)
          meta[i] = ((ia * TB + ib) << 16) | ((d0 - lod0) * c1 + (d1 - lod1));
      }
    }
  }

  double R[MT_S_PER_WARP][4][2];
#pragma unroll
  for (int i = 0; i < MT_S_PER_WARP; ++i)
#pragma unroll
    for (int s = 0; s < 4; ++s) R[i][s][0] = R[i][s][1] = 0.0;

  __syncthreads();
  if (a.coef == nullptr) form_w(c.W, wq, a, 0, i00, i10, e0lo, e0hi, tid);  // step-invariant

  const int nA = c.stiff ? 2 * MT_A : MT_A;
  for (int e2 = 0; e2 < K; ++e2) {
    if (a.coef != nullptr) form_w(c.W, wq, a, e2, i00, i10, e0lo, e0hi, tid);
    __syncthreads();
    // stage A: units (m-tile, type)
    for (int u = c.warp; u < nA; u += NW) {
      if (c.stiff) stage_a_unit(c, u >> 1, u & 1);
      else stage_a_unit(c, u, 0);
    }
    __syncthreads();
    // stage B: units (m-tile, ib half)
    if (c.warp < 2 * MT_B) {
      if (c.warp & 1) stage_b_unit<1>(c, c.warp >> 1);
      else stage_b_unit<0>(c, c.warp >> 1);
    }
    __syncthreads();
    // stage S + flush of the finished row e2
    switch (e2 & 3) {
      case 0: stage_s<0>(c, R, a, e2); flush<0>(c, R, meta, pb, pc, a, e2, N); break;
      case 1: stage_s<1>(c, R, a, e2); flush<1>(c, R, meta, pb, pc, a, e2, N); break;
      case 2: stage_s<2>(c, R, a, e2); flush<2>(c, R, meta, pb, pc, a, e2, N); break;
      default: stage_s<3>(c, R, a, e2); flush<3>(c, R, meta, pb, pc, a, e2, N); break;
    }
  }
  // rows K .. K+P-1 received their last contribution from element K-1
  for (int I2 = K; I2 < N; ++I2) flush_any(I2 & 3, c, R, meta, pb, pc, a, I2, N);
}

}  // namespace p3

int launch_gsf_p3(const GsfArgs& a0, cudaStream_t s) {
  GsfArgs a = a0;
  const int64_t N = (int64_t)a.K + p3::P;
  const int planes = a.plane_end - a.plane_begin;
  if (planes <= 0) return IGA_OK;
  const int tiles0 = (planes + p3::TA - 1) / p3::TA;
  a.tiles1 = (int)((N + p3::TB - 1) / p3::TB);
  const int64_t grid = (int64_t)tiles0 * a.tiles1;
  cudaError_t e = cudaFuncSetAttribute(p3::k_gsf3_p3, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)p3::SMEM_BYTES);
  if (e != cudaSuccess) return check_cuda(e, "gsf_p3 smem attr");
  p3::k_gsf3_p3<<<(unsigned)grid, p3::NT, p3::SMEM_BYTES, s>>>(a);
  return check_cuda(cudaGetLastError(), "gsf_p3 launch");
}

}  // namespace iga

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
constexpr int ROWV = NB * NB * NB;       // values of an interior CSR row (343)
constexpr int NT = 256;                  // threads (8 warps)
constexpr int NW = NT / 32;
constexpr int MT_A = NCOL / 8;           // 14
constexpr int MT_B = NA0 * Q / 8;        // 7
constexpr int MT_S = NCOMBO / 8;         // 49
constexpr int MT_S_PER_WARP = (MT_S + NW - 1) / NW;  // 7

// shared memory layout (doubles)
constexpr int OFF_W = 0;                                  // [LA*Q][WP]
constexpr int OFF_X = OFF_W + LA * Q * WP;                // [2][NA0][NCOL]
constexpr int OFF_Y = OFF_X + 2 * NA0 * NCOL;             // [2*Q][YP]
constexpr int OFF_BA = OFF_Y + 2 * Q * YP;                // [2 types][LA][2 nt][32]
constexpr int OFF_BB = OFF_BA + 2 * LA * 2 * 32;          // [2 prods][LB][2 nt][32]
constexpr int OFF_ST = OFF_BB + 2 * LB * 2 * 32;          // staging [TA*TB][ROWV]
constexpr int OFF_WQ = OFF_ST + TA * TB * ROWV;           // weights [Q]
constexpr int SMEM_DOUBLES = OFF_WQ + 8;
constexpr size_t SMEM_BYTES = SMEM_DOUBLES * sizeof(double);

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0,
                                     double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// element offset of column k = 2*nt + j (r = k) for destination index i = l + r - P
// to be inside [0, T): is any column of n-tile nt useful for window element l?
__host__ __device__ constexpr bool nt_useful(int l, int nt, int T) {
  return (l + 2 * nt - P >= 0 && l + 2 * nt - P < T) || (l + 2 * nt + 1 - P >= 0 && l + 2 * nt + 1 - P < T);
}

// B-fragment column mapping: lane (g, t) holds B[k=t][n=g]; column n of n-tile nt
// is the pair (r, s) = (2nt + (n&1), (r + (n>>1)) & 3).
__device__ __forceinline__ int bcol_r(int nt, int g) { return 2 * nt + (g & 1); }
__device__ __forceinline__ int bcol_s(int nt, int g) { return (bcol_r(nt, g) + (g >> 1)) & 3; }

template <int PHI>
__device__ __forceinline__ void stage_s_and_flush(double (&R)[MT_S_PER_WARP][4][2], const double* sm,
                                                  double* stage, const GsfArgs& a, int e2,
                                                  int warp, int g, int t, int lane, bool stiff,
                                                  bool smass) {
  // B fragments of element e2: Z0 = V V, Z1 = D D (+ V V for stiffness+mass)
  const double* V2 = a.V + (int64_t)e2 * M * Q;
  double b0[2], b1[2];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int r = bcol_r(nt, g), s = bcol_s(nt, g);
    const double vr = __ldg(V2 + r * Q + t), vs = __ldg(V2 + s * Q + t);
    b0[nt] = vr * vs;
    if (stiff) {
      const double* D2 = a.D + (int64_t)e2 * M * Q;
      double z = __ldg(D2 + r * Q + t) * __ldg(D2 + s * Q + t);
      if (smass) z += b0[nt];
      b1[nt] = z;
    } else {
      b1[nt] = 0.0;
    }
  }
  const double* Ys = sm + OFF_Y;
#pragma unroll
  for (int i = 0; i < MT_S_PER_WARP; ++i) {
    const int mt = warp + i * NW;
    if (mt < MT_S) {
      const double a0 = Ys[(0 * Q + t) * YP + mt * 8 + g];
      const double a1 = stiff ? Ys[(1 * Q + t) * YP + mt * 8 + g] : 0.0;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        double c0, c1;
        dmma(c0, c1, a0, b0[nt], 0.0, 0.0);
        if (stiff) dmma(c0, c1, a1, b1[nt], c0, c1);
        // column k = 2nt + j has r = k: destination row e2 + k -> slot (PHI + k) & 3
        const int k0 = 2 * nt, k1 = 2 * nt + 1;
        if (k0 < 4 - t) R[i][(PHI + k0) & 3][0] += c0; else R[i][(PHI + k0) & 3][1] += c0;
        if (k1 < 4 - t) R[i][(PHI + k1) & 3][0] += c1; else R[i][(PHI + k1) & 3][1] += c1;
      }
    }
  }
}

// Row e2 (slot SL) is complete: lanes put their values into the staging rows.
template <int SL>
__device__ __forceinline__ void flush_slot(double (&R)[MT_S_PER_WARP][4][2], double* stage,
                                           int I2, int i00, int i10, int64_t N, int warp, int g,
                                           int t) {
  const int lod2 = max(0, P - I2);
  const int c2 = (int)band_cnt(I2, P, N);
#pragma unroll
  for (int i = 0; i < MT_S_PER_WARP; ++i) {
    const int mt = warp + i * NW;
    if (mt < MT_S) {
      const int c = mt * 8 + g;
      const int d1 = c % NB, ib = (c / NB) % TB, a0 = c / (NB * TB);
      const int d0 = a0 % NB, ia = a0 / NB;
      const int I0 = i00 + ia, I1 = i10 + ib;
      const int lod0 = max(0, P - I0), lod1 = max(0, P - I1);
      const int c0 = (int)band_cnt(I0, P, N), c1 = (int)band_cnt(I1, P, N);
      const bool ok01 = d0 >= lod0 && d0 < lod0 + c0 && d1 >= lod1 && d1 < lod1 + c1;
      double* row = stage + (ia * TB + ib) * ROWV;
      const int base = ((d0 - lod0) * c1 + (d1 - lod1)) * c2;
      const int dh = P + t, dl = t - 1;
      if (ok01 && dh >= lod2 && dh < lod2 + c2) row[base + dh - lod2] = R[i][SL][0];
      if (ok01 && t > 0 && dl >= lod2 && dl < lod2 + c2) row[base + dl - lod2] = R[i][SL][1];
      R[i][SL][0] = 0.0;
      R[i][SL][1] = 0.0;
    }
  }
}

__device__ __forceinline__ void flush_dispatch(int sl, double (&R)[MT_S_PER_WARP][4][2],
                                               double* stage, int I2, int i00, int i10, int64_t N,
                                               int warp, int g, int t) {
  switch (sl) {
    case 0: flush_slot<0>(R, stage, I2, i00, i10, N, warp, g, t); break;
    case 1: flush_slot<1>(R, stage, I2, i00, i10, N, warp, g, t); break;
    case 2: flush_slot<2>(R, stage, I2, i00, i10, N, warp, g, t); break;
    default: flush_slot<3>(R, stage, I2, i00, i10, N, warp, g, t); break;
  }
}

// Coalesced copy of the finished rows (I0, I1, I2) of the tile to the CSR values.
__device__ __forceinline__ void store_rows(const double* stage, const GsfArgs& a, int I2, int i00,
                                           int i10, int64_t N, int tid) {
  const int64_t c2 = band_cnt(I2, P, N);
#pragma unroll
  for (int rc = 0; rc < TA * TB; ++rc) {
    const int ia = rc / TB, ib = rc % TB;
    const int64_t I0 = i00 + ia, I1 = i10 + ib;
    if (I0 >= a.plane_end || I1 >= N) continue;
    const int cnt = (int)(band_cnt(I0, P, N) * band_cnt(I1, P, N) * c2);
    double* dst = a.values + (rowptr3(I0, I1, I2, P, N) - a.base);
    const double* src = stage + rc * ROWV;
    for (int j = tid; j < cnt; j += NT) dst[j] = src[j];
  }
}

__global__ void __launch_bounds__(NT, 1) k_gsf3_p3(GsfArgs a) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  const int K = a.K;
  const int64_t N = (int64_t)K + P;
  const int tile0 = blockIdx.x / a.tiles1, tile1 = blockIdx.x % a.tiles1;
  const int i00 = a.plane_begin + tile0 * TA, i10 = tile1 * TB;
  const bool stiff = a.op != IGA_OP_MASS;
  const bool smass = a.op == IGA_OP_STIFFNESS_MASS;
  const int e0lo = max(a.el_begin, 0), e0hi = min(a.el_end, K);
  double* W = sm + OFF_W;
  double* X = sm + OFF_X;
  double* Ys = sm + OFF_Y;
  double* BA = sm + OFF_BA;
  double* BB = sm + OFF_BB;
  double* stage = sm + OFF_ST;
  double* wq = sm + OFF_WQ;

  // ---- constant B fragments of axes 0 and 1 (pair products of the window elements)
  for (int u = tid; u < 2 * LA * 2 * 32; u += NT) {
    const int ln = u & 31, nt = (u >> 5) & 1, la = (u >> 6) % LA, type = u / (64 * LA);
    const int gg = ln >> 2, tt = ln & 3;
    const int e0 = i00 - P + la;
    double v = 0.0;
    if (e0 >= 0 && e0 < K && (type == 0 || stiff)) {
      const double* T = (type == 0 ? a.V : a.D) + (int64_t)e0 * M * Q;
      v = T[bcol_r(nt, gg) * Q + tt] * T[bcol_s(nt, gg) * Q + tt];
    }
    BA[u] = v;
  }
  for (int u = tid; u < 2 * LB * 2 * 32; u += NT) {
    const int ln = u & 31, nt = (u >> 5) & 1, lb = (u >> 6) % LB, prod = u / (64 * LB);
    const int gg = ln >> 2, tt = ln & 3;
    const int e1 = i10 - P + lb;
    double v = 0.0;
    if (e1 >= 0 && e1 < K && (prod == 0 || stiff)) {
      const double* T = (prod == 0 ? a.V : a.D) + (int64_t)e1 * M * Q;
      v = T[bcol_r(nt, gg) * Q + tt] * T[bcol_s(nt, gg) * Q + tt];
    }
    BB[u] = v;
  }
  if (tid < Q) wq[tid] = a.weights[tid];

  double R[MT_S_PER_WARP][4][2];
#pragma unroll
  for (int i = 0; i < MT_S_PER_WARP; ++i)
#pragma unroll
    for (int s = 0; s < 4; ++s) R[i][s][0] = R[i][s][1] = 0.0;

  __syncthreads();

  for (int e2 = 0; e2 < K; ++e2) {
    // ---- W[(la,k0)][(g1,k2)] = c * w0 w1 w2 * jac on the CTA's slab of element column e2
    for (int u = tid; u < LA * Q * NCOL; u += NT) {
      const int row = u / NCOL, col = u - row * NCOL;
      const int la = row >> 2, k0 = row & 3;
      const int g1 = col >> 2, k2 = col & 3, lb = g1 >> 2, k1 = g1 & 3;
      const int e0 = i00 - P + la, e1 = i10 - P + lb;
      double w = 0.0;
      if (e0 >= e0lo && e0 < e0hi && e1 >= 0 && e1 < K) {
        const double c = a.coef ? __ldg(a.coef + (((int64_t)e0 * K + e1) * K + e2) * (Q * Q * Q) +
                                        (k0 * Q + k1) * Q + k2)
                                : a.coef_scalar;
        w = wq[k0] * wq[k1] * wq[k2] * a.jac * c;
      }
      W[row * WP + col] = w;
    }
    __syncthreads();

    // ---- stage A: contract axis 0; lanes own columns (g1,k2), accumulate X[type][ia][d0]
    for (int mt = warp; mt < MT_A; mt += NW) {
      double acc[2][TA][2];
#pragma unroll
      for (int ty = 0; ty < 2; ++ty)
#pragma unroll
        for (int ia = 0; ia < TA; ++ia) acc[ty][ia][0] = acc[ty][ia][1] = 0.0;
#pragma unroll
      for (int la = 0; la < LA; ++la) {
        const double av = W[(la * Q + t) * WP + mt * 8 + g];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          if (!nt_useful(la, nt, TA)) continue;
#pragma unroll
          for (int ty = 0; ty < 2; ++ty) {
            if (ty == 1 && !stiff) continue;
            double c0, c1;
            dmma(c0, c1, av, BA[((ty * LA + la) * 2 + nt) * 32 + lane], 0.0, 0.0);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int k = 2 * nt + j, ia = la + k - P;
              if (ia >= 0 && ia < TA) {
                const double c = j ? c1 : c0;
                if (k < 4 - t) acc[ty][ia][0] += c; else acc[ty][ia][1] += c;
              }
            }
          }
        }
      }
      const int col = mt * 8 + g;
#pragma unroll
      for (int ty = 0; ty < 2; ++ty) {
        if (ty == 1 && !stiff) continue;
#pragma unroll
        for (int ia = 0; ia < TA; ++ia) {
          X[(ty * NA0 + ia * NB + P + t) * NCOL + col] = acc[ty][ia][0];
          if (t > 0) X[(ty * NA0 + ia * NB + t - 1) * NCOL + col] = acc[ty][ia][1];
        }
      }
    }
    __syncthreads();

    // ---- stage B: contract axis 1; rows (a0, k2), accumulate Y_A / Y_B[(a0, ib, d1)][k2]
    if (warp < MT_B) {
      const int mt = warp;
      const int row = mt * 8 + g, a0 = row >> 2, k2 = row & 3;
      double yA[TB][2], yB[TB][2];
#pragma unroll
      for (int ib = 0; ib < TB; ++ib) yA[ib][0] = yA[ib][1] = yB[ib][0] = yB[ib][1] = 0.0;
#pragma unroll
      for (int lb = 0; lb < LB; ++lb) {
        const int xo = (lb * Q + t) * Q + k2;
        const double xv = X[(0 * NA0 + a0) * NCOL + xo];
        const double xd = stiff ? X[(1 * NA0 + a0) * NCOL + xo] : 0.0;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          if (!nt_useful(lb, nt, TB)) continue;
          const double vv = BB[((0 * LB + lb) * 2 + nt) * 32 + lane];
          double cA0, cA1, cB0 = 0.0, cB1 = 0.0;
          if (stiff) {
            const double dd = BB[((1 * LB + lb) * 2 + nt) * 32 + lane];
            dmma(cA0, cA1, xd, vv, 0.0, 0.0);
            dmma(cA0, cA1, xv, dd, cA0, cA1);
            dmma(cB0, cB1, xv, vv, 0.0, 0.0);
          } else {
            dmma(cA0, cA1, xv, vv, 0.0, 0.0);
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int k = 2 * nt + j, ib = lb + k - P;
            if (ib >= 0 && ib < TB) {
              const double ca = j ? cA1 : cA0, cb = j ? cB1 : cB0;
              if (k < 4 - t) { yA[ib][0] += ca; yB[ib][0] += cb; }
              else { yA[ib][1] += ca; yB[ib][1] += cb; }
            }
          }
        }
      }
#pragma unroll
      for (int ib = 0; ib < TB; ++ib) {
        const int ch = (a0 * TB + ib) * NB + P + t;
        Ys[(0 * Q + k2) * YP + ch] = yA[ib][0];
        if (stiff) Ys[(1 * Q + k2) * YP + ch] = yB[ib][0];
        if (t > 0) {
          const int cl = (a0 * TB + ib) * NB + t - 1;
          Ys[(0 * Q + k2) * YP + cl] = yA[ib][1];
          if (stiff) Ys[(1 * Q + k2) * YP + cl] = yB[ib][1];
        }
      }
    }
    __syncthreads();

    // ---- stage S: contract axis 2 within element e2 into the rolling rows; flush row e2
    switch (e2 & 3) {
      case 0: stage_s_and_flush<0>(R, sm, stage, a, e2, warp, g, t, lane, stiff, smass); break;
      case 1: stage_s_and_flush<1>(R, sm, stage, a, e2, warp, g, t, lane, stiff, smass); break;
      case 2: stage_s_and_flush<2>(R, sm, stage, a, e2, warp, g, t, lane, stiff, smass); break;
      default: stage_s_and_flush<3>(R, sm, stage, a, e2, warp, g, t, lane, stiff, smass); break;
    }
    flush_dispatch(e2 & 3, R, stage, e2, i00, i10, N, warp, g, t);
    __syncthreads();
    store_rows(stage, a, e2, i00, i10, N, tid);
    if (e2 == K - 1) {
      // rows K .. K+P-1 received their last contribution from element K-1
      for (int I2 = K; I2 < N; ++I2) {
        __syncthreads();
        flush_dispatch(I2 & 3, R, stage, I2, i00, i10, N, warp, g, t);
        __syncthreads();
        store_rows(stage, a, I2, i00, i10, N, tid);
      }
    }
  }
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

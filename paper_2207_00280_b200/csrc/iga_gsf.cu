// Assembled sum factorization (row-owner), generic in (p, q): the general-coefficient
// integrate+assemble kernel for every degree (k_gsf3_p3 specialises p=3, q=4 on DMMA).
//
// The global CSR value of rows I = (I0, I1, I2), J (I0 slowest, assembly.py:25)
//   S[I,J] = sum_e sum_k W_e(k) prod_d T_d[e_d](I_d - e_d, k_d) T_d[e_d](J_d - e_d, k_d)
// is the element-by-element Gauss quadrature of integrators.py:77-151 summed
// over the elements that support both I and J (assembly.py:80-82).  Sum
// factorization contracts one axis at a time (integrators.py:120-151); here
// every contraction also runs over the *elements* along its axis, so the
// inter-element (assembly) sum is folded into the contraction and each CSR
// value is produced exactly once, by one thread, in a fixed order: no atomics,
// no element matrices in HBM, bitwise reproducible.
//
// Decomposition (one CTA per tile of TA x TB rows along axes 0 and 1, streaming
// the elements e2 of the fastest axis, SURVEY.md §7.2 mapping of the paper's
// concurrency levels):
//   stage W : W[g0][g1][k2] = c * w w w * jac on the CTA's quadrature slab
//   stage A : X_T[i0][d0][g1][k2] = sum_{e0,k0} T(I0) T(J0) W      (axis 0)
//   stage B : Y_*[i0][d0][i1][d1][k2] = sum_{e1,k1} X . pair(axis 1)  (axis 1)
//   stage S : R[rows e2..e2+p][cols] += sum_k2 Y . pair(axis 2)     (axis 2)
// and the row e2 finishes after element e2: it is written, coalesced, in CSR
// order, and its rolling slot recycled for row e2+p+1.
//
// Each contraction is a small dense GEMM whose one operand is constant for the CTA
// (the pair products of the tile's element windows, PA / PB / Z) and is read as a
// warp-uniform shared-memory broadcast, while the other operand (one W column, one
// X row, one Y combo) sits in registers: an item = (column or row, group of outputs),
// items enumerated column-fastest so that every lane of a warp works on the same
// output (the broadcast) of a different column.  Invalid element/row combinations
// carry zero pair products, so the loops have no data-dependent bounds.
//
// Operators (T = value table V or derivative table D of each axis):
//   mass            : X_V, Y_M = X_V VV,             S += Y_M VV
//   stiffness       : X_V, X_D, Y_A = X_D VV + X_V DD, Y_B = X_V VV,
//                     S += Y_A VV + Y_B DD
//   stiffness+mass  : as stiffness with S += Y_A VV + Y_B (DD + VV)
#include <cstdlib>

#include "iga_args.cuh"
#include "iga_dispatch.cuh"

namespace iga {

constexpr int kGsfThreads = 512;

__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ constexpr int rup32(int a) { return cdiv(a, 32) * 32; }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int cmax(int a, int b) { return a > b ? a : b; }

template <int P, int Q, int TA, int TB, bool STIFF>
struct GsfShape {
  static constexpr int m = P + 1;
  static constexpr int NB = 2 * P + 1;  // band width
  static constexpr int LA = TA + P, LB = TB + P;  // element windows of the tile
  static constexpr int KA = LA * Q, KB = LB * Q;  // contraction lengths (elements x points)
  static constexpr int GC = KB * Q;               // stage-A columns (lb, k1, k2)
  static constexpr int NA0 = TA * NB, NB1 = TB * NB;
  static constexpr int NC = NA0 * NB1;            // (a0, b1) combos
  static constexpr int NR = NA0 * Q;              // stage-B rows (a0, k2)
  static constexpr int rowVals = NB * NB * NB;
  // stage A items: (column, group of AG outputs a0)
  static constexpr int GCp = rup32(GC);
  static constexpr int AG = cmax(1, cmin(NA0, cdiv(NA0 * GCp, kGsfThreads)));
  static constexpr int NGA = cdiv(NA0, AG);
  // stage B items: (row, group of BG outputs b1)
  static constexpr int NRp = rup32(NR);
  static constexpr int BG = cmax(1, cmin(NB1, cdiv(NB1 * NRp, kGsfThreads)));
  static constexpr int NGB = cdiv(NB1, BG);
  // stage S items: (combo, group of SG rows r)
  static constexpr int NCp = rup32(NC);
  static constexpr int SG = cmax(1, cmin(m, cdiv(m * NCp, kGsfThreads)));
  static constexpr int NGS = cdiv(m, SG);
  // shared memory (doubles); Y aliases W (W is dead after stage A)
  static constexpr int nW = KA * GC;
  static constexpr int nY = 2 * NC * Q;
  static constexpr int nWY = nW > nY ? nW : nY;
  static constexpr int nPA = 2 * NA0 * KA;
  static constexpr int nPB = 2 * NB1 * KB;
  static constexpr int nX = 2 * NA0 * GC;
  static constexpr int nZ = 2 * m * m * Q;
  static constexpr int nR = TA * TB * m * rowVals;
  static constexpr size_t doubles = (size_t)nWY + nPA + nPB + nX + nZ + nR;
  static constexpr size_t bytes = doubles * sizeof(double);
};

template <int P, int Q, int TA, int TB, bool STIFF>
__global__ void __launch_bounds__(kGsfThreads, P <= 2 ? 2 : 1) k_gsf3(GsfArgs a) {
  using S = GsfShape<P, Q, TA, TB, STIFF>;
  constexpr int m = S::m, NB = S::NB, LA = S::LA, LB = S::LB, KA = S::KA, KB = S::KB;
  constexpr int GC = S::GC, NA0 = S::NA0, NB1 = S::NB1, NC = S::NC, NR = S::NR;
  extern __shared__ double smem[];
  double* sW = smem;                                               // [KA][GC]
  double2* Y2 = reinterpret_cast<double2*>(smem);                  // [NC][Q] (aliases W)
  double2* PA2 = reinterpret_cast<double2*>(smem + S::nWY);        // [NA0][KA] (VV, DD)
  double2* PB2 = PA2 + NA0 * KA;                                   // [NB1][KB] (VV, DD)
  double2* X2 = PB2 + NB1 * KB;                                    // [NA0][KB][Q] (XV, XD)
  double2* Z2 = X2 + NA0 * GC;                                     // [m][m][Q] (VV, DD(+VV))
  double* R = reinterpret_cast<double*>(Z2 + m * m * Q);           // [TA*TB][m][rowVals]
  __shared__ int64_t rowoff[TA * TB];

  const int K = a.K;
  const int64_t N = (int64_t)K + P;
  const int tile = blockIdx.x / a.segs, seg = blockIdx.x % a.segs;
  const int tile0 = tile / a.tiles1, tile1 = tile % a.tiles1;
  const int i00 = a.plane_begin + tile0 * TA;  // first row plane of the tile (axis 0)
  const int i10 = tile1 * TB;                  // first row index along axis 1
  // element-column segment: rows I2 in [s0, s1) are written by this CTA, which streams
  // the elements [s0 - P, s1) that contribute to them (the first P recomputed as halo)
  const int s0 = seg * a.seg_len, s1 = min(K, s0 + a.seg_len);
  const int e_first = max(0, s0 - P);
  const int tid = threadIdx.x, nt = blockDim.x;
  const int e0lo = max(a.el_begin, 0), e0hi = min(a.el_end, K);  // slab, clipped to the mesh
  const double* V = a.V;
  const double* D = a.D;

  // ---- constant pair tables of the tile: PA (axis 0, slab-restricted), PB (axis 1)
  for (int t = tid; t < NA0 * KA; t += nt) {
    const int a0 = t / KA, kk = t % KA, la = kk / Q, k0 = kk % Q;
    const int I0 = i00 + a0 / NB, J0 = I0 - P + a0 % NB, e0 = i00 - P + la;
    const int r = I0 - e0, sidx = J0 - e0;
    double2 v = make_double2(0.0, 0.0);
    if (e0 >= e0lo && e0 < e0hi && r >= 0 && r <= P && sidx >= 0 && sidx <= P && J0 >= 0 && J0 < N) {
      const double* Te = V + (int64_t)e0 * m * Q;
      v.x = Te[r * Q + k0] * Te[sidx * Q + k0];
      if (STIFF) {
        const double* De = D + (int64_t)e0 * m * Q;
        v.y = De[r * Q + k0] * De[sidx * Q + k0];
      }
    }
    PA2[t] = v;
  }
  for (int t = tid; t < NB1 * KB; t += nt) {
    const int b1 = t / KB, kk = t % KB, lb = kk / Q, k1 = kk % Q;
    const int I1 = i10 + b1 / NB, J1 = I1 - P + b1 % NB, e1 = i10 - P + lb;
    const int r = I1 - e1, sidx = J1 - e1;
    double2 v = make_double2(0.0, 0.0);
    if (e1 >= 0 && e1 < K && r >= 0 && r <= P && sidx >= 0 && sidx <= P && J1 >= 0 && J1 < N) {
      const double* Te = V + (int64_t)e1 * m * Q;
      v.x = Te[r * Q + k1] * Te[sidx * Q + k1];
      if (STIFF) {
        const double* De = D + (int64_t)e1 * m * Q;
        v.y = De[r * Q + k1] * De[sidx * Q + k1];
      }
    }
    PB2[t] = v;
  }
  for (int t = tid; t < S::nR; t += nt) R[t] = 0.0;

  // coefficient of element column e2 for this thread's W entries, loaded one column ahead
  constexpr int WPT = cdiv(S::nW, kGsfThreads);
  auto load_coef = [&](int e2, double (&cv)[WPT]) {
#pragma unroll
    for (int i = 0; i < WPT; ++i) {
      const int t = tid + i * nt;
      cv[i] = a.coef_scalar;
      if (a.coef && t < S::nW && e2 < K) {
        const int kk = t / GC, col = t % GC;
        const int la = kk / Q, k0 = kk % Q, lb = col / (Q * Q), k1 = (col / Q) % Q, k2 = col % Q;
        const int e0 = i00 - P + la, e1 = i10 - P + lb;
        if (e0 >= 0 && e0 < K && e1 >= 0 && e1 < K)
          cv[i] = __ldg(a.coef + (((int64_t)e0 * K + e1) * K + e2) * (Q * Q * Q) + (k0 * Q + k1) * Q + k2);
      }
    }
  };
  double cv[WPT];
  load_coef(e_first, cv);
  // axis-2 pair products of element e2: the table entries are loaded one column ahead
  constexpr int ZPT = cdiv(m * m * Q, kGsfThreads);
  auto load_z = [&](int e2, double (&zv)[ZPT][4]) {
#pragma unroll
    for (int i = 0; i < ZPT; ++i) {
      const int t = tid + i * nt;
      zv[i][0] = zv[i][1] = zv[i][2] = zv[i][3] = 0.0;
      if (t < m * m * Q && e2 < K) {
        const int k = t % Q, sidx = (t / Q) % m, r = t / (Q * m);
        const double* V2 = V + (int64_t)e2 * m * Q;
        zv[i][0] = __ldg(V2 + r * Q + k);
        zv[i][1] = __ldg(V2 + sidx * Q + k);
        if (STIFF) {
          const double* D2 = D + (int64_t)e2 * m * Q;
          zv[i][2] = __ldg(D2 + r * Q + k);
          zv[i][3] = __ldg(D2 + sidx * Q + k);
        }
      }
    }
  };
  double zv[ZPT][4];
  load_z(e_first, zv);
  for (int e2 = e_first; e2 < s1; ++e2) {
    __syncthreads();  // previous column's stage S (reads Y, aliasing W) is done
    // ---- stage W: weights x coefficient, [(la,k0)][(lb,k1,k2)]; Z: axis-2 pair products
#pragma unroll
    for (int i = 0; i < WPT; ++i) {
      const int t = tid + i * nt;
      if (t < S::nW) {
        const int kk = t / GC, col = t % GC;
        const int k0 = kk % Q, k1 = (col / Q) % Q, k2 = col % Q;
        sW[t] = a.weights[k0] * a.weights[k1] * a.weights[k2] * a.jac * cv[i];
      }
    }
    load_coef(e2 + 1, cv);
#pragma unroll
    for (int i = 0; i < ZPT; ++i) {
      const int t = tid + i * nt;
      if (t < m * m * Q) {
        const double vv = zv[i][0] * zv[i][1];
        double dd = 0.0;
        if (STIFF) {
          dd = zv[i][2] * zv[i][3];
          if (a.op == IGA_OP_STIFFNESS_MASS) dd += vv;
        }
        Z2[t] = make_double2(vv, dd);
      }
    }
    load_z(e2 + 1, zv);
    __syncthreads();
    // ---- stage A (axis 0): X_T[a0][col] = sum_{(la,k0)} PA_T[a0][(la,k0)] W[(la,k0)][col]
    for (int it = tid; it < S::GCp * S::NGA; it += nt) {
      const int col = it % S::GCp, g = it / S::GCp;
      if (col < GC) {
        double w[KA];
#pragma unroll
        for (int kk = 0; kk < KA; ++kk) w[kk] = sW[kk * GC + col];
#pragma unroll
        for (int j = 0; j < S::AG; ++j) {
          const int a0 = g * S::AG + j;
          if (a0 < NA0) {
            const double2* pa = PA2 + a0 * KA;
            double xv = 0.0, xd = 0.0;
#pragma unroll
            for (int kk = 0; kk < KA; ++kk) {
              const double2 pp = pa[kk];
              xv += pp.x * w[kk];
              if (STIFF) xd += pp.y * w[kk];
            }
            X2[a0 * GC + col] = make_double2(xv, xd);
          }
        }
      }
    }
    __syncthreads();
    // ---- stage B (axis 1): per row (a0, k2), Y over b1:
    //   mass: Y = sum XV VV;  stiffness: YA = sum XV DD + XD VV, YB = sum XV VV
    for (int it = tid; it < S::NRp * S::NGB; it += nt) {
      const int row = it % S::NRp, g = it / S::NRp;
      if (row < NR) {
        const int a0 = row / Q, k2 = row % Q;
        // pass 1: XV against (VV, DD); pass 2 (stiffness): XD against VV into YA
        double xr[KB];
#pragma unroll
        for (int kk = 0; kk < KB; ++kk) xr[kk] = X2[a0 * GC + kk * Q + k2].x;
#pragma unroll
        for (int j = 0; j < S::BG; ++j) {
          const int b1 = g * S::BG + j;
          if (b1 < NB1) {
            const double2* pb = PB2 + b1 * KB;
            double ya = 0.0, yb = 0.0;
#pragma unroll
            for (int kk = 0; kk < KB; ++kk) {
              const double2 pp = pb[kk];
              if (STIFF) {
                ya += xr[kk] * pp.y;
                yb += xr[kk] * pp.x;
              } else {
                ya += xr[kk] * pp.x;
              }
            }
            Y2[(a0 * NB1 + b1) * Q + k2] = make_double2(ya, yb);
          }
        }
        if (STIFF) {
#pragma unroll
          for (int kk = 0; kk < KB; ++kk) xr[kk] = X2[a0 * GC + kk * Q + k2].y;
#pragma unroll
          for (int j = 0; j < S::BG; ++j) {
            const int b1 = g * S::BG + j;
            if (b1 < NB1) {
              const double2* pb = PB2 + b1 * KB;
              double ya = 0.0;
#pragma unroll
              for (int kk = 0; kk < KB; ++kk) ya += xr[kk] * pb[kk].x;
              Y2[(a0 * NB1 + b1) * Q + k2].x += ya;
            }
          }
        }
      }
    }
    __syncthreads();
    // ---- stage S (axis 2): rolling rows R[row e2 + r] += sum_k2 Y Z(r, s)
    for (int it = tid; it < S::NCp * S::NGS; it += nt) {
      const int c = it % S::NCp, g = it / S::NCp;
      if (c < NC) {
        const int a0 = c / NB1, b1 = c % NB1;
        const int ia = a0 / NB, d0 = a0 % NB, ib = b1 / NB, d1 = b1 % NB;
        double ya[Q], yb[Q];
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          const double2 y = Y2[c * Q + k];
          ya[k] = y.x;
          yb[k] = y.y;
        }
        double* Rc = R + (ia * TB + ib) * m * S::rowVals + (d0 * NB + d1) * NB;
#pragma unroll
        for (int j = 0; j < S::SG; ++j) {
          const int r = g * S::SG + j;
          if (r < m) {
            double* Rr = Rc + ((e2 + r) % m) * S::rowVals + P - r;
#pragma unroll
            for (int sidx = 0; sidx < m; ++sidx) {
              const double2* z = Z2 + (r * m + sidx) * Q;
              double acc = 0.0;
#pragma unroll
              for (int k = 0; k < Q; ++k) {
                const double2 zz = z[k];
                acc += ya[k] * zz.x;
                if (STIFF) acc += yb[k] * zz.y;
              }
              Rr[sidx] += acc;
            }
          }
        }
      }
    }
    __syncthreads();
    // ---- write the finished rows I2 = e2 (and the tail rows after the last element) of
    // this segment; every slot is cleared after use (halo rows I2 < s0 are dropped)
    const int last = (e2 == K - 1) ? (int)N - 1 : e2;
    for (int I2 = e2; I2 <= last; ++I2) {
      const int slot = I2 % m;
      const bool write = I2 >= s0;
      if (write && tid < TA * TB) {  // per-pencil row offsets (64-bit) for this row
        const int ia = tid / TB, ib = tid % TB;
        const int64_t I0 = i00 + ia, I1 = i10 + ib;
        rowoff[tid] = (I0 < a.plane_end && I1 < N) ? rowptr3(I0, I1, I2, P, N) - a.base : -1;
      }
      __syncthreads();
      const int lod2 = max(0, P - I2), c2 = (int)band_cnt(I2, P, N);
      for (int t = tid; t < TA * TB * S::rowVals; t += nt) {
        const int rc = t / S::rowVals, v = t - rc * S::rowVals;
        double* Rv = R + (rc * m + slot) * S::rowVals + v;
        if (write) {
          const int64_t off = rowoff[rc];
          const int ia = rc / TB, ib = rc - ia * TB;
          const int I0 = i00 + ia, I1 = i10 + ib;
          if (off >= 0) {
            if (I0 >= P && I0 < K && I1 >= P && I1 < K && lod2 == 0 && c2 == NB) {
              a.values[off + v] = *Rv;  // full band: CSR order is the R order
            } else {
              const int d2 = v % NB, d1 = (v / NB) % NB, d0 = v / (NB * NB);
              const int lod0 = max(0, P - I0), lod1 = max(0, P - I1);
              const int c0 = (int)band_cnt(I0, P, N), c1 = (int)band_cnt(I1, P, N);
              if (d0 >= lod0 && d0 < lod0 + c0 && d1 >= lod1 && d1 < lod1 + c1 && d2 >= lod2 &&
                  d2 < lod2 + c2)
                a.values[off + ((d0 - lod0) * c1 + (d1 - lod1)) * c2 + (d2 - lod2)] = *Rv;
            }
          }
        }
        *Rv = 0.0;
      }
      __syncthreads();
    }
  }
}

// tile sizes: the largest of (2,4), (2,2), (2,1), (1,1) whose shared memory fits
template <int P, int Q, bool ST>
struct GsfTile {
  static constexpr size_t cap = 227 * 1024;
  static constexpr int TA = GsfShape<P, Q, 2, 4, ST>::bytes <= cap ? 2
                            : GsfShape<P, Q, 2, 2, ST>::bytes <= cap ? 2
                            : GsfShape<P, Q, 2, 1, ST>::bytes <= cap ? 2 : 1;
  static constexpr int TB = GsfShape<P, Q, 2, 4, ST>::bytes <= cap ? 4
                            : GsfShape<P, Q, 2, 2, ST>::bytes <= cap ? 2 : 1;
};

int launch_gsf_p3(const GsfArgs& a, cudaStream_t s);   // iga_gsf_p3.cu (DMMA, p=3 q=4)
int launch_gsf_p3s(const GsfArgs& a, cudaStream_t s);  // iga_gsf_p3s.cu (symmetric, whole mesh)

// The symmetric-half kernels write S[I, J] and its mirror S[J, I] from one computation, valid
// when the call writes every row its element range touches: rows [el_begin, el_end + p) of
// the mesh (a whole mesh; a multi-GPU slab with its interface planes)
bool sym_covers(const GsfArgs& a, int p) {
  const int e0 = a.el_begin > 0 ? a.el_begin : 0, e1 = a.el_end < a.K ? a.el_end : a.K;
  const int last = e1 + p < a.K + p ? e1 + p : a.K + p;
  return e1 > e0 && a.plane_begin <= e0 && a.plane_end >= last;
}

// Before a symmetric launch on a slab (plane_begin > 0): the first p planes' rows hold values
// with J0 < plane_begin, which no element of the slab supports (they are 0) and which the
// symmetric kernels would only write as mirrors of rows outside the slab -- zero those rows
int sym_prezero(const GsfArgs& a, int p, cudaStream_t s) {
  if (a.plane_begin <= 0) return IGA_OK;
  const int64_t N = (int64_t)a.K + p;
  const int64_t hi = a.plane_begin + p < a.plane_end ? a.plane_begin + p : a.plane_end;
  const int64_t n = rowptr3(hi, 0, 0, p, N) - rowptr3(a.plane_begin, 0, 0, p, N);
  if (n > 0) return check_cuda(cudaMemsetAsync(a.values, 0, (size_t)n * sizeof(double), s), "slab prezero");
  return IGA_OK;
}

// A/B knobs: on only for the exact value "1", read once per process
static bool env_is_one(const char* name) {
  const char* e = getenv(name);
  return e != nullptr && e[0] == '1' && e[1] == 0;
}
int launch_gsf_mma(const GsfArgs& a, int p, int q, cudaStream_t s);  // iga_gsf_mma.cu (DMMA)
int launch_gsf_tile(const GsfArgs& a, int p, int q, cudaStream_t s);  // iga_tile.cu (p <= 2)
bool tile_wins(int p, int op);                                         // iga_tile.cu

template <int P, int Q, bool ST>
static int launch_gsf_generic(const GsfArgs& a0, cudaStream_t s) {
  constexpr int TA = GsfTile<P, Q, ST>::TA, TB = GsfTile<P, Q, ST>::TB;
  using Sh = GsfShape<P, Q, TA, TB, ST>;
  if constexpr (Sh::bytes > 227 * 1024) {
    set_error("assembled sum factorization: p=%d q=%d needs %zu B shared memory", P, Q, Sh::bytes);
    return IGA_EUNSUPPORTED;
  } else {
    GsfArgs a = a0;
    const int64_t N = (int64_t)a.K + P;
    const int planes = a.plane_end - a.plane_begin;
    if (planes <= 0) return IGA_OK;
    const int tiles0 = (planes + TA - 1) / TA;
    a.tiles1 = (int)((N + TB - 1) / TB);
    const int64_t tiles = (int64_t)tiles0 * a.tiles1;
    const void* fn = reinterpret_cast<const void*>(k_gsf3<P, Q, TA, TB, ST>);
    cudaError_t e = smem_attr_once(fn, Sh::bytes);
    if (e != cudaSuccess) return check_cuda(e, "gsf smem attr");
    // split the element column into segments when the tiles alone do not fill the GPU:
    // minimise waves x (segment + halo) element iterations
    const int64_t slots = (int64_t)sm_count() * blocks_per_sm_once(fn, kGsfThreads, Sh::bytes);
    int best = 1;
    double best_cost = 1e300;
    for (int sg = 1; sg <= a.K; ++sg) {
      const int L = (a.K + sg - 1) / sg;
      if (L < P && sg > 1) break;
      const int64_t ctas = tiles * sg;
      const double waves = (double)((ctas + slots - 1) / slots);
      const double cost = waves * (L + (sg > 1 ? P : 0));
      if (cost < best_cost - 1e-9) { best_cost = cost; best = sg; }
    }
    a.segs = best;
    a.seg_len = (a.K + best - 1) / best;
    k_gsf3<P, Q, TA, TB, ST><<<(unsigned)(tiles * best), kGsfThreads, Sh::bytes, s>>>(a);
    return check_cuda(cudaGetLastError(), "gsf launch");
  }
}

template <int P, int Q>
struct GsfLaunch {
  static int run(const GsfArgs& a0, cudaStream_t s) {
    if constexpr (P == 3 && Q == 4) {
      // tensor-core specialisation; IGA_GSF_GENERIC=1 selects the generic kernel (A/B tests)
      static const bool generic = env_is_one("IGA_GSF_GENERIC");
      // the symmetric variant computes J0 >= I0 and mirrors the rest, so the call must write
      // every row its elements touch (a whole mesh, or an element slab with its interface
      // planes); IGA_GSF_SYM=0 selects k_gsf3_p3 (A/B tests)
      static const bool no_sym = [] {
        const char* e = getenv("IGA_GSF_SYM");
        return e != nullptr && e[0] == '0' && e[1] == 0;
      }();
      if (!generic && sym_covers(a0, P) && !no_sym) {
        const int rc = sym_prezero(a0, P, s);
        return rc != IGA_OK ? rc : launch_gsf_p3s(a0, s);
      }
      if (!generic) return launch_gsf_p3(a0, s);
    }
    if constexpr (P >= 1 && P <= 2) {
      // non-streaming tile kernel where it is the faster one; IGA_GSF_TILE=0 / 1 forces the
      // streaming / tile kernels (A/B tests)
      static const int tile_env = [] {
        const char* e = getenv("IGA_GSF_TILE");
        return e == nullptr || e[0] == 0 || e[1] != 0 ? -1 : (e[0] == '0' ? 0 : (e[0] == '1' ? 1 : -1));
      }();
      if (tile_env == 1 || (tile_env == -1 && tile_wins(P, a0.op))) {
        const int rc = launch_gsf_tile(a0, P, Q, s);
        if (rc != IGA_EUNSUPPORTED) return rc;  // else: tile does not fit shared memory
      }
    }
    // DMMA GEMM formulation; IGA_GSF_SCALAR=1 selects this file's scalar kernel (A/B tests,
    // uniform knots only)
    static const bool scalar = env_is_one("IGA_GSF_SCALAR");
    if (!scalar || a0.wt != nullptr) return launch_gsf_mma(a0, P, Q, s);
    if (a0.op == IGA_OP_MASS) return launch_gsf_generic<P, Q, false>(a0, s);
    if constexpr (P >= 1) return launch_gsf_generic<P, Q, true>(a0, s);
    set_error("derivatives require degree >= 1");
    return IGA_EINVAL;
  }
};

int launch_gsf(const GsfArgs& a, int p, int q, cudaStream_t s) {
  return dispatch_pq<GsfLaunch>(p, q, a, s);
}

}  // namespace iga

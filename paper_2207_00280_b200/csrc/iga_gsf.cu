// Assembled sum factorization (row-owner): the headline integrate+assemble
// kernel.
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
// Operators (T = value table V or derivative table D of each axis):
//   mass            : X_V, Y_M = X_V VV,             S += Y_M VV
//   stiffness       : X_V, X_D, Y_A = X_D VV + X_V DD, Y_B = X_V VV,
//                     S += Y_A VV + Y_B DD
//   stiffness+mass  : as stiffness with S += Y_A VV + Y_B (DD + VV)
#include <cstdlib>

#include "iga_args.cuh"
#include "iga_dispatch.cuh"

namespace iga {

template <int P, int Q, int TA, int TB>
struct GsfShape {
  static constexpr int m = P + 1;
  static constexpr int NB = 2 * P + 1;                 // band width
  static constexpr int GA = (TA + P) * Q;              // quadrature points on axis 0 slab
  static constexpr int GB = (TB + P) * Q;              // ... axis 1
  static constexpr int nW = GA * GB * Q;
  static constexpr int nTabA = (TA + P) * m * Q;
  static constexpr int nTabB = (TB + P) * m * Q;
  static constexpr int nX = TA * NB * GB * Q;          // per type
  static constexpr int nCombo = TA * NB * TB * NB;
  static constexpr int nY = nCombo * Q;                // per accumulator
  static constexpr int rowVals = NB * NB * NB;
  static constexpr int nR = TA * TB * m * rowVals;
  static constexpr int nZ = m * m * Q;
  static constexpr size_t doubles = (size_t)nW + 2 * nTabA + 2 * nTabB + 2 * nX + 2 * nY + nR + 2 * nZ;
  static constexpr size_t bytes = doubles * sizeof(double);
};

template <int P, int Q, int TA, int TB>
__global__ void __launch_bounds__(512, 2) k_gsf3(GsfArgs a) {
  using S = GsfShape<P, Q, TA, TB>;
  constexpr int m = S::m, NB = S::NB, GB = S::GB;
  extern __shared__ double smem[];
  double* sW = smem;
  double* tAV = sW + S::nW;
  double* tAD = tAV + S::nTabA;
  double* tBV = tAD + S::nTabA;
  double* tBD = tBV + S::nTabB;
  double* XV = tBD + S::nTabB;
  double* XD = XV + S::nX;
  double* Y0 = XD + S::nX;
  double* Y1 = Y0 + S::nY;
  double* R = Y1 + S::nY;
  double* Z0 = R + S::nR;
  double* Z1 = Z0 + S::nZ;
  __shared__ int64_t rowoff[TA * TB];

  const int K = a.K;
  const int64_t N = (int64_t)K + P;
  const int tile = blockIdx.x / a.segs, seg = blockIdx.x % a.segs;
  const int tile0 = tile / a.tiles1, tile1 = tile % a.tiles1;
  const int i00 = a.plane_begin + tile0 * TA;  // first row plane of the tile (axis 0)
  // element-column segment: rows I2 in [s0, s1) are written by this CTA, which streams
  // the elements [s0 - P, s1) that contribute to them (the first P recomputed as halo)
  const int s0 = seg * a.seg_len, s1 = min(K, s0 + a.seg_len);
  const int e_first = max(0, s0 - P);
  const int i10 = tile1 * TB;                  // first row index along axis 1
  const int tid = threadIdx.x, nt = blockDim.x;
  const bool stiff = a.op != IGA_OP_MASS;
  const int e0lo = max(a.el_begin, 0), e0hi = min(a.el_end, K);  // slab, clipped to the mesh

  // per-axis tables of the CTA's element windows (zero outside the mesh)
  for (int t = tid; t < S::nTabA; t += nt) {
    const int e = i00 - P + t / (m * Q);
    const bool ok = e >= 0 && e < K;
    tAV[t] = ok ? a.V[(int64_t)e * m * Q + t % (m * Q)] : 0.0;
    tAD[t] = ok && stiff ? a.D[(int64_t)e * m * Q + t % (m * Q)] : 0.0;
  }
  for (int t = tid; t < S::nTabB; t += nt) {
    const int e = i10 - P + t / (m * Q);
    const bool ok = e >= 0 && e < K;
    tBV[t] = ok ? a.V[(int64_t)e * m * Q + t % (m * Q)] : 0.0;
    tBD[t] = ok && stiff ? a.D[(int64_t)e * m * Q + t % (m * Q)] : 0.0;
  }
  for (int t = tid; t < S::nR; t += nt) R[t] = 0.0;

  // coefficient of element column e2 for this thread's W entries (loaded one column
  // ahead, so the global-memory latency overlaps the previous column's stages)
  constexpr int WPT = (S::nW + 511) / 512;
  auto load_coef = [&](int e2, double (&cv)[WPT]) {
#pragma unroll
    for (int i = 0; i < WPT; ++i) {
      const int t = tid + i * nt;
      cv[i] = a.coef_scalar;
      if (a.coef && t < S::nW && e2 < K) {
        const int k2 = t % Q, g1 = (t / Q) % GB, g0 = t / (Q * GB);
        const int la = g0 / Q, k0 = g0 % Q, lb = g1 / Q, k1 = g1 % Q;
        const int e0 = i00 - P + la, e1 = i10 - P + lb;
        if (e0 >= e0lo && e0 < e0hi && e1 >= 0 && e1 < K)
          cv[i] = __ldg(a.coef + (((int64_t)e0 * K + e1) * K + e2) * (Q * Q * Q) + (k0 * Q + k1) * Q + k2);
      }
    }
  };
  double cv[WPT];
  load_coef(e_first, cv);
  for (int e2 = e_first; e2 < s1; ++e2) {
    __syncthreads();
    // ---- stage W: weights x coefficient on the (axis0, axis1) slab of element column e2
#pragma unroll
    for (int i = 0; i < WPT; ++i) {
      const int t = tid + i * nt;
      if (t < S::nW) {
        const int k2 = t % Q, g1 = (t / Q) % GB, g0 = t / (Q * GB);
        const int la = g0 / Q, k0 = g0 % Q, lb = g1 / Q, k1 = g1 % Q;
        const int e0 = i00 - P + la, e1 = i10 - P + lb;
        double W = 0.0;
        if (e0 >= e0lo && e0 < e0hi && e1 >= 0 && e1 < K)
          W = a.weights[k0] * a.weights[k1] * a.weights[k2] * a.jac * cv[i];
        sW[t] = W;
      }
    }
    load_coef(e2 + 1, cv);
    // pair tables of axis 2 for element e2: Z0 = VV, Z1 = DD (+VV)
    for (int t = tid; t < S::nZ; t += nt) {
      const int k = t % Q, s = (t / Q) % m, r = t / (Q * m);
      const double* V2 = a.V + (int64_t)e2 * m * Q;
      const double vv = V2[r * Q + k] * V2[s * Q + k];
      Z0[t] = vv;
      if (stiff) {
        const double* D2 = a.D + (int64_t)e2 * m * Q;
        double dd = D2[r * Q + k] * D2[s * Q + k];
        if (a.op == IGA_OP_STIFFNESS_MASS) dd += vv;
        Z1[t] = dd;
      }
    }
    __syncthreads();
    // ---- stage A: contract axis 0 (elements e0 and points k0)
    for (int t = tid; t < S::nX; t += nt) {
      const int k2 = t % Q;
      const int g1 = (t / Q) % GB;
      const int d0 = (t / (Q * GB)) % NB;
      const int ia = t / (Q * GB * NB);
      const int I0 = i00 + ia, J0 = I0 - P + d0;
      const int lo = max(max(I0, J0) - P, 0), hi = min(min(I0, J0), K - 1);
      double xv = 0.0, xd = 0.0;
      for (int e0 = lo; e0 <= hi; ++e0) {
        const int la = e0 - (i00 - P);
        const double* av = tAV + la * m * Q;
        const double* ad = tAD + la * m * Q;
        const int r = I0 - e0, s = J0 - e0;
#pragma unroll
        for (int k0 = 0; k0 < Q; ++k0) {
          const double W = sW[((la * Q + k0) * GB + g1) * Q + k2];
          xv += av[r * Q + k0] * av[s * Q + k0] * W;
          if (stiff) xd += ad[r * Q + k0] * ad[s * Q + k0] * W;
        }
      }
      XV[t] = xv;
      XD[t] = xd;
    }
    __syncthreads();
    // ---- stage B: contract axis 1 (elements e1 and points k1)
    for (int t = tid; t < S::nY; t += nt) {
      const int k2 = t % Q;
      const int d1 = (t / Q) % NB;
      const int ib = (t / (Q * NB)) % TB;
      const int a0 = t / (Q * NB * TB);  // = ia * NB + d0
      const int I1 = i10 + ib, J1 = I1 - P + d1;
      const int lo = max(max(I1, J1) - P, 0), hi = min(min(I1, J1), K - 1);
      double y0 = 0.0, y1 = 0.0;
      for (int e1 = lo; e1 <= hi; ++e1) {
        const int lb = e1 - (i10 - P);
        const double* bv = tBV + lb * m * Q;
        const double* bd = tBD + lb * m * Q;
        const int r = I1 - e1, s = J1 - e1;
#pragma unroll
        for (int k1 = 0; k1 < Q; ++k1) {
          const int xi = (a0 * GB + lb * Q + k1) * Q + k2;
          const double vv = bv[r * Q + k1] * bv[s * Q + k1];
          if (stiff) {
            const double dd = bd[r * Q + k1] * bd[s * Q + k1];
            y0 += XD[xi] * vv + XV[xi] * dd;
            y1 += XV[xi] * vv;
          } else {
            y0 += XV[xi] * vv;
          }
        }
      }
      Y0[t] = y0;
      Y1[t] = y1;
    }
    __syncthreads();
    // ---- stage S: contract axis 2 within element e2 into the rolling rows
    for (int t = tid; t < S::nCombo * m * m; t += nt) {
      const int s = t % m;
      const int r = (t / m) % m;
      const int c = t / (m * m);  // ((ia*NB + d0)*TB + ib)*NB + d1
      const int d1 = c % NB, ib = (c / NB) % TB, d0 = (c / (NB * TB)) % NB, ia = c / (NB * TB * NB);
      const double* y0 = Y0 + c * Q;
      const double* y1 = Y1 + c * Q;
      const double* z0 = Z0 + (r * m + s) * Q;
      const double* z1 = Z1 + (r * m + s) * Q;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < Q; ++k) {
        acc += y0[k] * z0[k];
        if (stiff) acc += y1[k] * z1[k];
      }
      const int slot = (e2 + r) % m;
      const int d2 = s - r + P;
      R[(((ia * TB + ib) * m + slot) * NB + d0) * NB * NB + d1 * NB + d2] += acc;
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
        const int rc = t / S::rowVals, v = t % S::rowVals;
        const int d2 = v % NB, d1 = (v / NB) % NB, d0 = v / (NB * NB);
        double* Rv = R + (rc * m + slot) * S::rowVals + v;
        if (write) {
          const int64_t off = rowoff[rc];
          const int ia = rc / TB, ib = rc % TB;
          const int I0 = i00 + ia, I1 = i10 + ib;
          const int lod0 = max(0, P - I0), lod1 = max(0, P - I1);
          const int c0 = (int)band_cnt(I0, P, N), c1 = (int)band_cnt(I1, P, N);
          if (off >= 0 && d0 >= lod0 && d0 < lod0 + c0 && d1 >= lod1 && d1 < lod1 + c1 &&
              d2 >= lod2 && d2 < lod2 + c2)
            a.values[off + ((d0 - lod0) * c1 + (d1 - lod1)) * c2 + (d2 - lod2)] = *Rv;
        }
        *Rv = 0.0;
      }
      __syncthreads();
    }
  }
}

template <int P>
struct GsfTile {
  // tile sizes keep the shared-memory footprint under 227 KB
  static constexpr int TA = P <= 3 ? 2 : (P == 4 ? 2 : 1);
  static constexpr int TB = P <= 3 ? 4 : (P == 4 ? 2 : 1);
};

int launch_gsf_p3(const GsfArgs& a, cudaStream_t s);  // iga_gsf_p3.cu (DMMA, p=3 q=4)

template <int P, int Q>
struct GsfLaunch {
  static int run(const GsfArgs& a0, cudaStream_t s) {
    if constexpr (P == 3 && Q == 4) {
      // tensor-core specialisation; IGA_GSF_GENERIC=1 selects the generic kernel (A/B tests)
      const char* env = getenv("IGA_GSF_GENERIC");
      if (!(env && env[0] == '1')) return launch_gsf_p3(a0, s);
    }
    constexpr int TA = GsfTile<P>::TA, TB = GsfTile<P>::TB;
    using Sh = GsfShape<P, Q, TA, TB>;
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
      const void* fn = reinterpret_cast<const void*>(k_gsf3<P, Q, TA, TB>);
      cudaError_t e = smem_attr_once(fn, Sh::bytes);
      if (e != cudaSuccess) return check_cuda(e, "gsf smem attr");
      // split the element column into segments when the tiles alone do not fill the GPU:
      // minimise waves x (segment + halo) element iterations
      const int64_t slots = (int64_t)sm_count() * blocks_per_sm_once(fn, 512, Sh::bytes);
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
      k_gsf3<P, Q, TA, TB><<<(unsigned)(tiles * best), 512, Sh::bytes, s>>>(a);
      return check_cuda(cudaGetLastError(), "gsf launch");
    }
  }
};

int launch_gsf(const GsfArgs& a, int p, int q, cudaStream_t s) {
  return dispatch_pq<GsfLaunch>(p, q, a, s);
}

}  // namespace iga

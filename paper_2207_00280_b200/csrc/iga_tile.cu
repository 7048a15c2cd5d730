// Assembled sum factorization for low degrees (1 <= p <= 2) without streaming: one CTA per
// TA x TB x TC tile of rows (I0, I1, I2), and the three contractions of the reference's
// sum factorization (integrators.py:112-151) run over the tile's element window
// [I - p, I + T) per axis, assembly included (assembly.py:80-82):
//
//   stage A (axis 0): X_T[(ia,d0)][g1][g2] = sum_{g0} PA_T[(ia,d0)][g0] W[g0][g1][g2]
//   stage B (axis 1): Y[(ia,d0)][(ib,d1)][g2] = sum_{g1} X[(ia,d0)][g1][g2] PB[(ib,d1)][g1]
//   stage S (axis 2): S[(ia,ib,ic)][(d0,d1,d2)] = sum_{g2} Y[(ia,d0)][(ib,d1)][g2] PC[(ic,d2)][g2]
//
// g = (l, k): window element l and Gauss point k of an axis; (i, d): tile row i and band
// offset d (column J = I - p + d).  P?[(i,d)][(l,k)] = T(I - e, k) T(J - e, k) w_k is
// nonzero only where the element e = base + l supports both dofs, a compile-time band
// l in [i + max(0, d - p), i + min(p, d)]: every contraction is a fully unrolled DFMA
// sequence over exactly its nonzero terms, and a thread keeps the band rows of its tile
// index in registers (stage_band).  The quadrature weights (and the Jacobian) are folded
// into the P tables, so W is the coefficient field itself, copied into shared memory by
// one 3D TMA box (zero outside the mesh or the element slab; cp.async where TMA cannot
// describe the window).  CTAs are persistent, each over a contiguous range of tiles.
//
// Why a second kernel for p <= 2: the streaming kernels (k_gsf3_mma, iga_gsf_mma.cu) pay
// per element column four CTA barriers, a row flush, the pair-table setup of a short
// segment and DMMA tiles that are mostly padding at these sizes; on C2 (32^3, p = 2 mass
// with a coefficient field) that was ~680 warp instructions per row, instruction-issue
// bound at 9% of the HBM roofline.  Here a tile costs ~4 barriers, each thread works on
// whole vectors of one stage with operands in registers, and two CTAs per SM overlap one
// tile's coefficient copy with the other's arithmetic.  The window recomputation
// ((T + p) / T per axis) costs flops, which these degrees have to spare.  Dispatch:
// tile_wins() below.  Summation order is fixed (bitwise reproducible).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <type_traits>

#include "iga_args.cuh"
#include "iga_dispatch.cuh"

namespace iga {
namespace tile {

__host__ __device__ constexpr int imax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int imin(int a, int b) { return a < b ? a : b; }

constexpr int NT = 256;


template <int P, int Q, int TA, int TB, int TC, bool ST>
struct Shape {
  static constexpr int NB = 2 * P + 1, m = P + 1, E = ST ? 2 : 1;
  static constexpr int LA = TA + P, LB = TB + P, LC = TC + P;
  static constexpr int GA = LA * Q, GB = LB * Q, GC = LC * Q;
  static constexpr int RA = TA * NB, RB = TB * NB, RC = TC * NB;
  static constexpr int GCY = GC | 1;  // Y row pitch: odd, stage-S row loads conflict-free
  // pair-table rows padded to an even length (16-byte aligned rows; the pad is 0)
  static constexpr int GAP = (GA + 1) / 2 * 2, GBP = (GB + 1) / 2 * 2, GCP = (GC + 1) / 2 * 2;
  static constexpr int nW = GA * GB * GC;
  static constexpr int nX = (E * RA * GB * GC + 1) / 2 * 2;
  static constexpr int nY = E * RA * RB * GCY;
  static constexpr int nR1 = (imax(nW, nY) + 1) / 2 * 2;  // W, then Y (W dead after stage A)
  static constexpr int nPA = E * RA * GAP, nPB = E * RB * GBP, nPC = E * RC * GCP;
  static constexpr int nRows = TA * TB * TC;
  static constexpr int nE = ((LA + LB + LC) * (2 * m + 1) * Q + 1) / 2 * 2;  // element records
  // doubles; the int64 row bases and int band info follow
  static constexpr int nD = nR1 + nX + nPA + nPB + nPC + nE;
  static constexpr int ER = (2 * m + 1) * Q;  // doubles of an element record (V, D, w)
  static constexpr size_t bytes = sizeof(double) * nD + sizeof(int64_t) * (nRows + TA * TB) +
                                  sizeof(int) * (4 * TA * TB + 2 * TC);
  // the mesh's element records cached once per CTA after that, for K <= kall(): within the
  // shared memory of the kernel's two CTAs per SM (or one, for the shapes that need more)
  // (228 KB per SM hold two CTAs of <= 111 KB dynamic + the static and reserved 1 KB each)
  static constexpr size_t lim = bytes <= 111 * 1024 ? 111 * 1024 : 225 * 1024;
  static constexpr size_t eall_off = (bytes + 15) / 16 * 16;
  static constexpr int kall() { return lim > eall_off ? (int)((lim - eall_off) / (ER * sizeof(double))) : 0; }
};

// first / one-past-last window element of band row (i, d) (element l supports tile row i
// and column offset d)
template <int P>
__host__ __device__ constexpr int band_l0(int i, int d) { return i + imax(0, d - P); }
template <int P>
__host__ __device__ constexpr int band_l1(int i, int d) { return i + imin(P, d) + 1; }

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}

// Element records of the three windows, staged once per CTA (one round of independent
// global loads) so the pair tables are built from shared memory: record of window element
// l of an axis = [V: m q][D: m q][w: q], zero for elements outside the mesh (or slab)
template <int P, int Q>
__host__ __device__ constexpr int erec() { return (2 * (P + 1) + 1) * Q; }

template <int P, int Q, int L>
__device__ __forceinline__ void stage_elements(double* Er, int first, int elo, int ehi, const GsfArgs& a, int tid) {
  constexpr int m = P + 1, ER = erec<P, Q>();
  for (int u = tid; u < L * ER; u += NT) {
    const int l = u / ER, j = u - l * ER, e = first + l;
    double val = 0.0;
    if (e >= elo && e < ehi) {
      if (j < m * Q) val = __ldg(a.V + (int64_t)e * m * Q + j);
      else if (j < 2 * m * Q) val = a.D != nullptr ? __ldg(a.D + (int64_t)e * m * Q + j - m * Q) : 0.0;
      else val = axis_w(a.weights, a.wt, e, j - 2 * m * Q, Q);
    }
    Er[u] = val;
  }
}

// Pair table of one axis: Pt[t][(i,d)][(l,k)] for the tile rows I = i0 + i, element e = i0 - P + l
// read from the records Er[e - ebase] where e is in [elo, ehi) (else 0), with the axis weight (and
// `scale`) folded in; type 1 = derivative products, plus the value products if `addv`
// (stiffness + mass, axis 2).
template <int P, int Q, int T, int E>
__device__ __forceinline__ void pair_table(double* Pt, const double* Er, int ebase, int elo, int ehi, int i0, int N,
                                           double scale, bool addv, int tid) {
  constexpr int NB = 2 * P + 1, m = P + 1, G = (T + P) * Q, GP = (G + 1) / 2 * 2, R = T * NB;
  constexpr int ER = erec<P, Q>();
  for (int u = tid; u < E * R * GP; u += NT) {
    const int ty = u / (R * GP), rem = u - ty * R * GP, row = rem / GP, g = rem - row * GP;
    const int i = row / NB, d = row - i * NB, l = g / Q, k = g - l * Q;
    const int J = i0 + i - P + d;
    const int r = P + i - l, s = i + d - l;  // I - e, J - e
    double v = 0.0;
    const int e = i0 - P + l;
    if (g < G && r >= 0 && r <= P && s >= 0 && s <= P && J >= 0 && J < N && e >= elo && e < ehi) {
      const double* rec = Er + (e - ebase) * ER;
      const double w = rec[2 * m * Q + k] * scale;  // 0 outside the mesh / slab
      const double vv = rec[r * Q + k] * rec[s * Q + k];
      if (ty == 0) {
        v = vv * w;
      } else {
        double dd = rec[m * Q + r * Q + k] * rec[m * Q + s * Q + k];
        if (addv) dd += vv;
        v = dd * w;
      }
    }
    Pt[u] = v;
  }
}

// 3D TMA copy of the coefficient window into shared memory, completing on an mbarrier
__device__ __forceinline__ void tma_load_3d(double* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            uint64_t* bar, unsigned bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst), b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(d),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(b)
      : "memory");
}

// One contraction stage.  Tile index i of the axis (T of them) gets NT / T threads; a thread
// loads the band rows (i, d) of its i for the d of chunk `ch` (of NSPL) from the pair
// table(s) into registers, then for each of its vectors u (of NV) loads the (p+1) q
// operand entries its i touches (element window i .. i+p: load(u, i, v)) and stores the
// 2p+1 (chunk) outputs row = i (2p+1) + d (store(u, row, x, y)).
//   one type (TWO = false): x = sum P v
//   two types (TWO): x = sum P0 v1 + P1 v0, y = sum P0 v0 (v0 = load, v1 = load2): the
//   stiffness products Y_A = X_D PB_V + X_V PB_D, Y_B = X_V PB_V (load = X_V, load2 = X_D)
//   and, with y unused, S = Y_A PC_V + Y_B PC_D (load = Y_B, load2 = Y_A)
template <int P, int Q, int T, int NSPL, bool TWO, class LD, class STO, class LD2>
__device__ __forceinline__ void stage_band(int tid, int ch, int NV, const double* P0, int pitch0, const double* P1,
                                           int pitch1, LD&& load, STO&& store, LD2&& load2) {
  constexpr int NB = 2 * P + 1, G = (P + 1) * Q, TPI = NT / T;
  static_assert(NT % T == 0, "threads split evenly over the tile indices");
  constexpr int DCH = (NB + NSPL - 1) / NSPL;
  const int i = tid / TPI, sub = tid - i * TPI;
  const int d0 = ch * DCH, d1 = d0 + DCH < NB ? d0 + DCH : NB;
  // band of row (i, d) relative to the union [i Q, (i + P + 1) Q): [max(0, d-P) Q, (min(P, d) + 1) Q)
  double p0[DCH][G], p1[TWO ? DCH : 1][TWO ? G : 1];
#pragma unroll
  for (int dd = 0; dd < DCH; ++dd) {
    const int d = d0 + dd;
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const bool in = d < d1 && j >= imax(0, d - P) * Q && j < (imin(P, d) + 1) * Q;
      p0[dd][j] = in ? P0[(i * NB + d) * pitch0 + i * Q + j] : 0.0;
      if constexpr (TWO) p1[dd][j] = in ? P1[(i * NB + d) * pitch1 + i * Q + j] : 0.0;
    }
  }
  auto sweep = [&](int u, const double (&v)[G], const double (&w)[TWO ? G : 1]) {
#pragma unroll
    for (int dd = 0; dd < DCH; ++dd) {
      const int d = d0 + dd;
      if (d >= d1) break;
      double x = 0.0, y = 0.0;
#pragma unroll
      for (int j = 0; j < G; ++j) {
        if (j < imax(0, d - P) * Q || j >= (imin(P, d) + 1) * Q) continue;  // outside the band
        if constexpr (TWO) {
          x = fma(p0[dd][j], w[j], x);
          x = fma(p1[dd][j], v[j], x);
          y = fma(p0[dd][j], v[j], y);
        } else {
          x = fma(p0[dd][j], v[j], x);
        }
      }
      store(u, i * NB + d, x, y);
    }
  };
  {
    // load(u) precedes the stores of u (callers may set per-vector store context in load)
    for (int u = sub; u < NV; u += TPI) {
      double v[G], w[TWO ? G : 1];
      load(u, i, v);
      if constexpr (TWO) load2(u, i, w);
      sweep(u, v, w);
    }
  }
}

template <int P, int Q, int TA, int TB, int TC, bool ST>
__global__ void __launch_bounds__(NT, 2)
    k_tile3(GsfArgs a, const __grid_constant__ CUtensorMap tm, int use_tma, int ntiles, int eall) {
  using S = Shape<P, Q, TA, TB, TC, ST>;
  constexpr int NB = S::NB, LA = S::LA, LB = S::LB, LC = S::LC;
  constexpr int GB = S::GB, GC = S::GC, GCY = S::GCY;
  constexpr int RA = S::RA, RB = S::RB, Q3 = Q * Q * Q, ER = erec<P, Q>();
  extern __shared__ __align__(128) double sm[];
  double* W = sm;               // [LA][LB][LC][Q^3] (element-major)
  double* Y = sm;               // [E][RA][RB][GCY] (aliases W)
  double* X = sm + S::nR1;      // [E][RA][GB][GC]
  double* PA = X + S::nX;       // [E][RA][GAP]
  double* PB = PA + S::nPA;     // [E][RB][GBP]
  double* PC = PB + S::nPB;     // [E][RC][GCP]
  double* EA = PC + S::nPC;     // element records of the three windows [LA | LB | LC][ER]
  double* EB = EA + LA * ER;
  double* EC = EB + LB * ER;
  int64_t* rowb = reinterpret_cast<int64_t*>(EA + S::nE);  // [TA][TB][TC]
  int64_t* base01 = rowb + S::nRows;                         // [TA*TB] CSR offset of row (I0, I1, 0)
  int* bnd01 = reinterpret_cast<int*>(base01 + TA * TB);    // [TA*TB][lod0, c0, lod1, c1]
  int* bnd2 = bnd01 + 4 * TA * TB;                            // [TC][lod2, c2]
  double* EALL = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + S::eall_off);  // [K][ER] if eall
  __shared__ uint64_t wbar;

  const int K = a.K, N = K + P, tid = threadIdx.x;
  const int tiles2 = (N + TC - 1) / TC;
  const int e0lo = max(a.el_begin, 0), e0hi = min(a.el_end, K);
  const unsigned wbar_s = (unsigned)__cvta_generic_to_shared(&wbar);
  if (use_tma && tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(wbar_s) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }

  if (eall) {
    // every element record of the mesh, once (the windows below then read shared memory)
    for (int u = tid; u < K * ER; u += NT) {
      const int e = u / ER, j = u - e * ER;
      constexpr int m = P + 1;
      double val;
      if (j < m * Q) val = __ldg(a.V + (int64_t)e * m * Q + j);
      else if (j < 2 * m * Q) val = a.D != nullptr ? __ldg(a.D + (int64_t)e * m * Q + j - m * Q) : 0.0;
      else val = axis_w(a.weights, a.wt, e, j - 2 * m * Q, Q);
      EALL[u] = val;
    }
    __syncthreads();
  }

  // Persistent CTAs (one wave), each taking a contiguous range of tiles (t2 fastest): a pair
  // table depends only on its axis' tile index and is rebuilt only when that index changes,
  // so consecutive tiles of a range share PA / PB.
  int h0 = -1, h1 = -1, h2 = -1;  // axis tile indices of the tables held
  int it = 0;
  const int per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int tbeg = blockIdx.x * per, tend = min(ntiles, tbeg + per);
  for (int tile = tbeg; tile < tend; ++tile, ++it) {
    const int t01 = tile / tiles2, t2 = tile - t01 * tiles2;
    const int t0 = t01 / a.tiles1, t1 = t01 - t0 * a.tiles1;
    const int i0 = a.plane_begin + t0 * TA, i1 = t1 * TB, i2 = t2 * TC;
    const bool n0 = t0 != h0, n1 = t1 != h1, n2 = t2 != h2;
    h0 = t0;
    h1 = t1;
    h2 = t2;
    if (it > 0) __syncthreads();  // the previous tile's stage S is done with Y (= W), X, tables

    // ---- coefficient window, element-major like the coefficient array: W[la][lb][lc][q^3]
    // (zero outside the mesh / slab)
    if (use_tma) {
      // one TMA box [LA][LB][LC q^3] of the tensor [slab e0][K e1][K q^3]: out-of-range
      // elements (mesh edges, other slabs) arrive as zeros
      if (tid == 0) tma_load_3d(W, &tm, (i2 - P) * Q3, i1 - P, i0 - P - e0lo, &wbar, (unsigned)(S::nW * sizeof(double)));
    } else {
      // word by word (cp.async): the LC q^3 coefficients of one (e0, e1) pair are contiguous
      // in memory and in W, thread j of a segment copies word j of every pair
      constexpr int SEG = LC * Q3, SPP = NT / SEG > 0 ? NT / SEG : 1;  // segments per pass
      const int sj = tid % SEG, sp = tid / SEG;
      const int e2 = i2 - P + sj / Q3;
      const bool ok2 = e2 >= 0 && e2 < K;
      const int64_t sK = (int64_t)K * Q3, sKK = sK * K;
      const double* src0 = a.coef + ((int64_t)(i0 - P) * K + (i1 - P)) * sK + (int64_t)(i2 - P) * Q3 + sj;
      if (sp < SPP) {
#pragma unroll
        for (int la = 0; la < LA; ++la) {
          const int e0 = i0 - P + la;
          const bool ok0 = ok2 && e0 >= e0lo && e0 < e0hi;
          for (int lb = sp; lb < LB; lb += SPP) {
            const int e1 = i1 - P + lb;
            const bool ok = ok0 && e1 >= 0 && e1 < K;
            double* dst = W + (la * LB + lb) * SEG + sj;
            if (a.coef) cp_async8(dst, ok ? src0 + la * sKK + lb * sK : a.coef, ok);
            else *dst = ok ? a.coef_scalar : 0.0;
          }
        }
      }
      if constexpr (SEG > NT) {
        // segments longer than the CTA (large q): the rest of each segment
        for (int lab = 0; lab < LA * LB; ++lab) {
          const int la = lab / LB, lb = lab - la * LB;
          const int e0 = i0 - P + la, e1 = i1 - P + lb;
          for (int j = NT + tid; j < SEG; j += NT) {
            const int e2j = i2 - P + j / Q3;
            const bool ok = e0 >= e0lo && e0 < e0hi && e1 >= 0 && e1 < K && e2j >= 0 && e2j < K;
            double* dst = W + lab * SEG + j;
            if (a.coef) cp_async8(dst, ok ? src0 - sj + la * sKK + lb * sK + j : a.coef, ok);
            else *dst = ok ? a.coef_scalar : 0.0;
          }
        }
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }

    // ---- pair tables of the changed axes (weights folded; the Jacobian on axis 2)
    constexpr int BIG = 0x7fffffff;
    if (eall) {
      if (n0) pair_table<P, Q, TA, S::E>(PA, EALL, 0, e0lo, e0hi, i0, N, 1.0, false, tid);
      if (n1) pair_table<P, Q, TB, S::E>(PB, EALL, 0, 0, K, i1, N, 1.0, false, tid);
      if (n2) pair_table<P, Q, TC, S::E>(PC, EALL, 0, 0, K, i2, N, a.jac, a.op == IGA_OP_STIFFNESS_MASS, tid);
    } else {
      if (n0) stage_elements<P, Q, LA>(EA, i0 - P, e0lo, e0hi, a, tid);
      if (n1) stage_elements<P, Q, LB>(EB, i1 - P, 0, K, a, tid);
      if (n2) stage_elements<P, Q, LC>(EC, i2 - P, 0, K, a, tid);
      __syncthreads();
      if (n0) pair_table<P, Q, TA, S::E>(PA, EA, i0 - P, -BIG, BIG, i0, N, 1.0, false, tid);
      if (n1) pair_table<P, Q, TB, S::E>(PB, EB, i1 - P, -BIG, BIG, i1, N, 1.0, false, tid);
      if (n2)
        pair_table<P, Q, TC, S::E>(PC, EC, i2 - P, -BIG, BIG, i2, N, a.jac, a.op == IGA_OP_STIFFNESS_MASS, tid);
    }
    // ---- the tile's CSR rows: row (I0, I1, I2) = row (I0, I1, 0) + c0 c1 band_prefix(I2)
    if (n0 || n1) {
      for (int u = tid; u < TA * TB; u += NT) {
        const int I0 = i0 + u / TB, I1 = i1 + u % TB;
        base01[u] = I0 < a.plane_end && I0 < N && I1 < N ? rowptr3(I0, I1, 0, P, N) - a.base : -1;
      }
      __syncthreads();
    }
    for (int u = tid; u < S::nRows; u += NT) {
      const int pc = u / TC, ic = u - pc * TC;
      const int I0 = i0 + pc / TB, I1 = i1 + pc % TB, I2 = i2 + ic;
      const int64_t b = base01[pc];
      rowb[u] = b >= 0 && I2 < N ? b + band_cnt(I0, P, N) * band_cnt(I1, P, N) * band_prefix(I2, P, N) : -1;
    }
    if (n0 || n1) {
      for (int u = tid; u < TA * TB; u += NT) {
        const int I0 = i0 + u / TB, I1 = i1 + u % TB;
        bnd01[4 * u + 0] = max(0, P - I0);
        bnd01[4 * u + 1] = I0 < N ? (int)band_cnt(I0, P, N) : 0;
        bnd01[4 * u + 2] = max(0, P - I1);
        bnd01[4 * u + 3] = I1 < N ? (int)band_cnt(I1, P, N) : 0;
      }
    }
    if (n2) {
      for (int u = tid; u < TC; u += NT) {
        const int I2 = i2 + u;
        bnd2[2 * u + 0] = max(0, P - I2);
        bnd2[2 * u + 1] = I2 < N ? (int)band_cnt(I2, P, N) : 0;
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    if (use_tma) {
      asm volatile(
          "{\n .reg .pred p;\n"
          "TW%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          " @!p bra TW%=;\n}\n" ::"r"(wbar_s),
          "r"(it & 1)
          : "memory");
    }

  // Every stage: the CTA's threads are split evenly over the tile indices i of the stage's
  // axis; a thread keeps the band rows (i, d), d < 2p+1, of its i in registers (RowBand:
  // 27 values for p = 2, q = 3) and sweeps its share of the stage's vectors, loading the
  // (p+1) q entries of each vector its i touches once and accumulating the 2p+1 outputs in
  // independent registers.  Stiffness splits the rows into two chunks so that both operand
  // types fit the registers.
  constexpr int NSPL = ST ? (P >= 2 ? 3 : 2) : 1;

  // ---- stage A: vectors = the (g1, g2) columns of W; outputs X_T[(ia, d0)][column]
  {
    auto load_w = [&](int c, int i, double (&v)[(P + 1) * Q]) {
      const int g1 = c / GC, g2 = c - g1 * GC, lb = g1 / Q, k1 = g1 - lb * Q, lc = g2 / Q, k2 = g2 - lc * Q;
      const double* wc = W + (i * LB * LC + lb * LC + lc) * Q3 + k1 * Q + k2;  // element la = i
#pragma unroll
      for (int j = 0; j < (P + 1) * Q; ++j) v[j] = wc[(j / Q) * LB * LC * Q3 + (j % Q) * Q * Q];
    };
    for (int ty = 0; ty < S::E; ++ty)
      stage_band<P, Q, TA, 1, false>(
          tid, 0, GB * GC, PA + ty * RA * S::GAP, S::GAP, nullptr, 0, load_w,
          [&](int c, int row, double x, double) { X[(ty * RA + row) * GB * GC + c] = x; }, load_w);
  }
  __syncthreads();

  // ---- stage B: vectors = the ((ia,d0), g2) rows of X; mass: Y = X_V PB_V; stiffness:
  // Y_A = X_D PB_V + X_V PB_D, Y_B = X_V PB_V
  for (int ch = 0; ch < NSPL; ++ch)
    stage_band<P, Q, TB, NSPL, ST>(
        tid, ch, RA * GC, PB, S::GBP, ST ? PB + RB * S::GBP : nullptr, S::GBP,
        [&](int u, int i, double (&v)[(P + 1) * Q]) {
          const int a0 = u / GC, g2 = u - a0 * GC;
          const double* xc = X + (a0 * GB + i * Q) * GC + g2;
#pragma unroll
          for (int j = 0; j < (P + 1) * Q; ++j) v[j] = xc[j * GC];
        },
        [&](int u, int row, double ya, double yb) {
          const int a0 = u / GC, g2 = u - a0 * GC;
          Y[(a0 * RB + row) * GCY + g2] = ya;
          if constexpr (ST) Y[((RA + a0) * RB + row) * GCY + g2] = yb;
        },
        [&](int u, int i, double (&v)[(P + 1) * Q]) {  // second operand type (X_D)
          const int a0 = u / GC, g2 = u - a0 * GC;
          const double* xc = X + ((RA + a0) * GB + i * Q) * GC + g2;
#pragma unroll
          for (int j = 0; j < (P + 1) * Q; ++j) v[j] = xc[j * GC];
        });
  __syncthreads();

  // ---- stage S: vectors = the ((ia,d0), (ib,d1)) rows of Y; the outputs go straight to the
  // CSR.  Each thread keeps one (I0, I1) pencil of its row ic = i (TPP threads per pencil,
  // taking its (d0, d1) blocks TPP apart), so the pencil's row base and band bounds are read
  // once per stage instead of per vector.  (Assembling a pencil's rows in shared memory and
  // writing contiguous runs measured 25% slower on C2: the extra barrier and copy loop cost
  // more than the 2p+1-value block stores.)
  {
    constexpr int TPI = NT / TC, NPEN = TA * TB, TPP = TPI / NPEN, NBLK = NB * NB;
    static_assert(TPI % NPEN == 0 && TPP >= 1, "threads split evenly over the pencils");
    constexpr int KV = (NBLK + TPP - 1) / TPP;  // blocks per thread (the last may be partial)
    const int ic = tid / TPI, sub = tid - ic * TPI, pen = sub / TPP, bsub = sub - pen * TPP;
    const int ia = pen / TB, ib = pen - ia * TB;
    const int lod0 = bnd01[4 * pen], c0 = bnd01[4 * pen + 1], lod1 = bnd01[4 * pen + 2],
              c1 = bnd01[4 * pen + 3];
    const int lod2 = bnd2[2 * ic], c2 = bnd2[2 * ic + 1];
    const int64_t rb = rowb[pen * TC + ic];
    int64_t gbase = 0;     // CSR offset of the current block in row ic, minus lod2
    int slo = 0, shi = 0;  // its valid d2 range [slo, shi) (empty: outside the band / mesh)
    int yrow = 0;          // its Y row (ia, d0) x (ib, d1)
    // vector j of stage_band = the thread's (j / TPI)-th block
    auto sctx = [&](int j) {
      const int blk = bsub + (j / TPI) * TPP;
      const int d0 = blk / NB, d1 = blk - d0 * NB;
      slo = shi = 0;
      yrow = blk < NBLK ? (ia * NB + d0) * RB + ib * NB + d1 : 0;
      if (blk < NBLK && rb >= 0 && d0 >= lod0 && d0 < lod0 + c0 && d1 >= lod1 && d1 < lod1 + c1) {
        gbase = rb + (int64_t)((d0 - lod0) * c1 + (d1 - lod1)) * c2 - lod2;
        slo = lod2;
        shi = lod2 + c2;
      }
    };
    for (int ch = 0; ch < NSPL; ++ch)
      stage_band<P, Q, TC, NSPL, ST>(
          tid, ch, TPI * KV, PC, S::GCP, ST ? PC + S::RC * S::GCP : nullptr, S::GCP,
          [&](int j, int i, double (&v)[(P + 1) * Q]) {
            sctx(j);
            const double* yc = Y + ((ST ? RA * RB : 0) + yrow) * GCY + i * Q;  // Y_B (stiffness) / Y
#pragma unroll
            for (int k = 0; k < (P + 1) * Q; ++k) v[k] = yc[k];
          },
          [&](int, int row, double x, double) {
            const int d2 = row % NB;
            if (d2 >= slo && d2 < shi) a.values[gbase + d2] = x;
          },
          [&](int, int i, double (&v)[(P + 1) * Q]) {  // second operand type (Y_A), same block
            const double* yc = Y + yrow * GCY + i * Q;
#pragma unroll
            for (int k = 0; k < (P + 1) * Q; ++k) v[k] = yc[k];
          });
  }
  }  // tiles
}

// Tile per degree: p = 2 mass 4 x 4 x 2 (80 KB, two CTAs per SM), p = 2 stiffness 4 x 2 x 2
// (97 KB), p = 1 8 x 4 x 4 / 4 x 4 x 4 (fewer window recomputations at the same footprint)
template <int P, int Q, bool ST>
struct Tile {
  static constexpr int TA = P == 1 ? (ST ? 4 : 8) : 4;
  static constexpr int TB = P == 1 ? 4 : (ST ? 2 : 4);
  static constexpr int TC = P == 1 ? 4 : 2;
};

// Tensor map of the coefficient field as [slab e0][K e1][K q^3] doubles with box
// [LA][LB][LC q^3]; false where TMA cannot describe it (inner box > 256 elements or not a
// multiple of 16 bytes, row strides not multiples of 16 bytes), and the kernel then copies
// word by word with cp.async
static bool coef_tensor_map(CUtensorMap& tm, const GsfArgs& a, int q3, int LA, int LB, int LC) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  const int64_t K = a.K, e0lo = a.el_begin > 0 ? a.el_begin : 0, e0hi = a.el_end < a.K ? a.el_end : a.K;
  const int64_t inner = (int64_t)LC * q3;
  const double* base = a.coef + e0lo * K * K * q3;
  if (encode == nullptr || e0hi <= e0lo || inner > 256 || (inner * 8) % 16 != 0 || (K * q3 * 8) % 16 != 0 ||
      reinterpret_cast<uintptr_t>(base) % 16 != 0)
    return false;
  const cuuint64_t dims[3] = {(cuuint64_t)(K * q3), (cuuint64_t)K, (cuuint64_t)(e0hi - e0lo)};
  const cuuint64_t strides[2] = {(cuuint64_t)(K * q3 * 8), (cuuint64_t)(K * K * q3 * 8)};
  const cuuint32_t box[3] = {(cuuint32_t)inner, (cuuint32_t)LB, (cuuint32_t)LA};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int P, int Q, bool ST>
static int launch_t(const GsfArgs& a0, cudaStream_t s) {
  constexpr int TA = Tile<P, Q, ST>::TA, TB = Tile<P, Q, ST>::TB, TC = Tile<P, Q, ST>::TC;
  using Sh = Shape<P, Q, TA, TB, TC, ST>;
  if constexpr (Sh::bytes > 227 * 1024) {
    return IGA_EUNSUPPORTED;  // the caller takes the streaming kernel
  } else {
    GsfArgs a = a0;
    const int64_t N = (int64_t)a.K + P;
    const int planes = a.plane_end - a.plane_begin;
    if (planes <= 0) return IGA_OK;
    const int64_t tiles0 = (planes + TA - 1) / TA;
    a.tiles1 = (int)((N + TB - 1) / TB);
    const int64_t grid = tiles0 * a.tiles1 * ((N + TC - 1) / TC);
    if (grid > 0x7fffffffLL) {
      set_error("tile sum factorization: %lld tiles exceed the grid limit", (long long)grid);
      return IGA_EUNSUPPORTED;
    }
    const void* fn = reinterpret_cast<const void*>(k_tile3<P, Q, TA, TB, TC, ST>);
    cudaError_t e = smem_attr_once(fn, Sh::lim, true);
    if (e != cudaSuccess) return check_cuda(e, "tile smem attr");
    CUtensorMap tm{};
    const int use_tma = a.coef != nullptr && coef_tensor_map(tm, a, Q * Q * Q, Sh::LA, Sh::LB, Sh::LC);
    const int64_t slots = (int64_t)sm_count() * blocks_per_sm_once(fn, NT, Sh::bytes);
    const int64_t ctas = grid < slots ? grid : slots;
    const int eall = a.K <= Sh::kall();
    const size_t smem = eall ? Sh::eall_off + (size_t)a.K * Sh::ER * sizeof(double) : Sh::bytes;
    k_tile3<P, Q, TA, TB, TC, ST><<<(unsigned)ctas, NT, smem, s>>>(a, tm, use_tma, (int)grid, eall);
    return check_cuda(cudaGetLastError(), "tile launch");
  }
}

}  // namespace tile

// The operators where the tile kernel beats the streaming kernels (tools/tile_shapes.py, one
// B200; kernel + K1 step time, tile vs streaming): p = 2 mass (32^3 0.053 vs 0.064 ms, 64^3
// 0.27 vs 0.31, 128^3 1.91 vs 1.97), p = 1 mass and stiffness (64^3 0.068 vs 0.123, 0.123 vs
// 0.162).  For p = 2 stiffness its two-type stages are 2-2.5x slower than the DMMA kernel
// (64^3 1.09 vs 0.42 ms): three contractions per stage on scalar FMAs.
bool tile_wins(int p, int op) { return p == 1 || (p == 2 && op == IGA_OP_MASS); }

// p in {1, 2}, q <= p + 3 (the shapes of iga_dispatch.cuh); returns IGA_EUNSUPPORTED for
// the rest, which the caller serves with the streaming kernels
int launch_gsf_tile(const GsfArgs& a, int p, int q, cudaStream_t s) {
#define IGA_TILE_CASE(PP, QQ)                                                          \
  if (p == PP && q == QQ) {                                                            \
    if (a.op == IGA_OP_MASS) return tile::launch_t<PP, QQ, false>(a, s);               \
    return tile::launch_t<PP, QQ, true>(a, s);                                         \
  }
  IGA_TILE_CASE(1, 1) IGA_TILE_CASE(1, 2) IGA_TILE_CASE(1, 3) IGA_TILE_CASE(1, 4)
  IGA_TILE_CASE(2, 1) IGA_TILE_CASE(2, 2) IGA_TILE_CASE(2, 3) IGA_TILE_CASE(2, 4) IGA_TILE_CASE(2, 5)
#undef IGA_TILE_CASE
  return IGA_EUNSUPPORTED;
}

}  // namespace iga

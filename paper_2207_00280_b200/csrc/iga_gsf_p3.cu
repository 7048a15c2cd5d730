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
// to the assembled values in registers -- no shared-memory read-modify-write,
// no atomics, and a fixed summation order (bitwise reproducible).
//
//   stage A (axis 0): C[(g1,k2)][(r,s)] = sum_k0 W[la,k0][(g1,k2)] PA_la[k0][(r,s)]
//                     -> X_T[ia = la+r-3][d0][(g1,k2)]                (T = V, D)
//   stage B (axis 1): C[(a0,k2)][(r,s)] = sum_k1 X_T[a0][(lb,k1,k2)] PB_lb[k1][(r,s)]
//                     -> Y_A/Y_B[(a0, ib = lb+r-3, d1)][k2]
//   stage S (axis 2): C[c][(r,s)] = sum_k2 Y[c][k2] Z_e2[k2][(r,s)]
//                     -> R[c][row e2+r][d2]  (rolling over 4 rows)
//
// Warp specialisation (software pipeline over the element column e2): 4 warps
// run stage A on element e2 = it, 4 warps stage B on e2 = it-1 and 8 warps stage
// S (+ the row stores) on e2 = it-2, all concurrently (512 threads x 128
// registers).  X and Y are double-buffered and handed from role to role by
// shared-memory mbarriers (full / empty per buffer), so no role waits for the
// whole CTA.  The DMMA pipe of every SM sub-partition is shared by the three
// stages and stays busy across what would otherwise be barrier-separated phases.
// The constant B fragments of stages A and B live in registers; the rolling rows
// of stage S live in per-lane shared-memory slots that are the DMMA C operands,
// and a row leaves for the CSR straight from the register of its last product.
#include <type_traits>

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
constexpr int XP = NCOL + 4;             // X row pitch (== 4 mod 16: conflict-free A stores)
constexpr int NA0 = TA * NB;             // (ia, d0) rows (14)
constexpr int NCOMBO = NA0 * TB * NB;    // (ia, d0, ib, d1) combos (392)
constexpr int YP = NCOMBO + 4;           // Y pitch (== 12 mod 16: conflict-free A loads)
constexpr int MT_A = NCOL / 8;           // 14 m-tiles of (g1,k2) columns
constexpr int MT_B = NA0 * Q / 8;        // 7 m-tiles of (a0,k2) rows
constexpr int MT_S = NCOMBO / 8;         // 49 m-tiles of combos
#ifndef P3_NWB
#define P3_NWB 5
#endif
#ifndef P3_BT
#define P3_BT 1
#endif
#ifndef P3_NWS
#define P3_NWS 7
#endif
#ifndef P3_NWA
#define P3_NWA 4
#endif
constexpr int NWA = P3_NWA, NWB = P3_NWB, NWS = P3_NWS;  // warps per role (NWA even: fixed type per A warp)
static_assert(NWA % 2 == 0, "stage-A warps come in (value, derivative) pairs");
constexpr int NT = 32 * (NWA + NWB + NWS);  // threads (16 warps by default)
constexpr int MT_S_PER_WARP = (MT_S + NWS - 1) / NWS;  // 7
constexpr int NHB = 2 * MT_B;            // stage-B half units (m-tile, ib pair)
constexpr int NPEN = TA * TB;            // row pencils (I0, I1) of the tile

// shared memory layout (doubles)
constexpr int SZ_X = 2 * NA0 * XP;                // one X buffer: [2 types][NA0][XP]
constexpr int SZ_Y = 2 * Q * YP;                  // one Y buffer: [2 accs * Q][YP]
constexpr int OFF_W = 0;                          // [LA*Q][WP]
constexpr int OFF_X = OFF_W + LA * Q * WP;        // 2 buffers
constexpr int OFF_Y = OFF_X + 2 * SZ_X;           // 2 buffers
// the constant B fragments are read into registers before the pipeline starts, so
// they alias Y buffer 1 (first written by stage B at iteration 2)
constexpr int OFF_BA = OFF_Y + SZ_Y;              // [2 types][LA pairs][32]
constexpr int OFF_BB = OFF_BA + 2 * LA * 32;      // [2 prods][10 pairs][32]
static_assert(2 * LA * 32 + 2 * 10 * 32 <= SZ_Y, "fragment tables fit Y buffer 1");
constexpr int OFF_WQ = OFF_Y + 2 * SZ_Y;          // weights [Q]
constexpr int OFF_PB = OFF_WQ + Q;                // pencil row-pointer bases (int64) [NPEN]
constexpr int OFF_PC = OFF_PB + NPEN;             // pencil c0*c1 (int in double slots) [NPEN]
constexpr int OFF_R = OFF_PC + NPEN;              // rolling rows [MT_S][4 slots][2 groups][32]
// axis-2 band table {band_prefix(I2), band_cnt(I2)} for meshes with N <= NBT rows (else computed)
constexpr int NBT = 1024;
constexpr int OFF_BT = OFF_R + MT_S * 4 * 2 * 32;  // int2 [NBT]
constexpr int OFF_MB = OFF_BT + (P3_BT ? NBT : 0);  // mbarriers [xfull 2][xempty 2][yfull 2][yempty 2]
constexpr int SMEM_DOUBLES = OFF_MB + 8;
static_assert(SMEM_DOUBLES * 8 <= 227 * 1024, "shared memory budget");
constexpr size_t SMEM_BYTES = SMEM_DOUBLES * sizeof(double);

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0,
                                     double c1) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
      : "=d"(d0), "=d"(d1)
      : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// shared-memory mbarriers: the roles hand buffers to each other (full / empty per
// buffer) instead of a CTA-wide barrier per element column
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "MBW%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MBW%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__host__ __device__ constexpr int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// B-fragment column mapping: lane (g, t) holds B[k=t][n=g]; column n of n-tile nt
// is the pair (r, s) = (2nt + (n&1), (r + (n>>1)) & 3).
__device__ __forceinline__ int bcol_r(int nt, int g) { return 2 * nt + (g & 1); }
__device__ __forceinline__ int bcol_s(int nt, int g) { return (bcol_r(nt, g) + (g >> 1)) & 3; }

// r += c on lanes where p holds (one predicated DADD, no select sequence)
__device__ __forceinline__ void add_if(double& r, double c, int p) {
  asm("{\n .reg .pred q;\n setp.ne.s32 q, %2, 0;\n @q add.rn.f64 %0, %0, %1;\n}\n"
      : "+d"(r)
      : "d"(c), "r"(p));
}

struct Lane {
  int lane, g, t;
  bool stiff, smass;
};

// hi = sum_{k < 4-t} y[k] (band offset 3+t), lo = sum of the rest (offset t-1)
// Lane masks m_k = [k < 4-t] as exact 0/1 doubles: fma(m, y, acc) adds y or nothing
// exactly, so the group sums need no data-dependent selects.
#ifndef P3_SPLIT
#define P3_SPLIT 0
#endif

__device__ __forceinline__ double sel(bool c, double a, double b) { return c ? a : b; }
__device__ __forceinline__ void split_groups(const double* y, int t, double& hi, double& lo) {
#if P3_SPLIT == 2
  // ablation only (wrong values): two DADDs instead of the six FP64 ops
  hi = y[0] + y[2];
  lo = y[1] + y[3];
#elif P3_SPLIT == 1
  // three DADDs per lane and integer selects: A = y0 + y1, B = y2 + y3, and one lane-chosen
  // sum C (t=0: A + B, t=1: A + y2, t=3: y1 + B)
  const double A = y[0] + y[1], B = y[2] + y[3];
  const double C = sel(t == 3, y[1], A) + sel(t == 1, y[2], B);
  hi = sel(t <= 1, C, sel(t == 2, A, y[0]));
  lo = sel(t == 1, y[3], sel(t == 2, B, C));
#else
  const double m1 = t <= 2 ? 1.0 : 0.0, m2 = t <= 1 ? 1.0 : 0.0, m3 = t == 0 ? 1.0 : 0.0;
  hi = fma(m3, y[3], fma(m2, y[2], fma(m1, y[1], y[0])));
  lo = fma(1.0 - m3, y[3], fma(1.0 - m2, y[2], (1.0 - m1) * y[1]));
#endif
}

// ---------------------------------------------------------------- stage A
// Stage-A B fragments pair two consecutive r = rb, rb+1 of one window element la;
// rb is chosen per la so that the 8 useful (la, r) combos (destination ia = la + r - P
// in [0, TA)) need 5 DMMAs per unit instead of 6 with fixed r-pairs.
constexpr int NPA = 5;
__host__ __device__ constexpr int pa_la(int i) { return i; }
__host__ __device__ constexpr int pa_rb(int i) { return i == 0 ? 2 : (i == 1 ? 2 : (i == 2 ? 1 : 0)); }

// NU units = m-tiles mt0 + i*mstep of (g1,k2) columns for the warp's type, interleaved
// for ILP; ba[] are the warp's constant B fragments; per-column accumulators
// acc[u][ia][r] are the DMMA C operands (each receives exactly one element's product).
template <int NU>
__device__ __forceinline__ void stage_a_units(const Lane& L, const double* W, const double (&ba)[NPA],
                                              double* X, int mt0, int mstep, int ty) {
  double acc[NU][TA][4];
#pragma unroll
  for (int u = 0; u < NU; ++u)
#pragma unroll
    for (int ia = 0; ia < TA; ++ia)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[u][ia][k] = 0.0;
  double av[NU][LA];
#pragma unroll
  for (int u = 0; u < NU; ++u)
#pragma unroll
    for (int la = 0; la < LA; ++la) av[u][la] = W[(la * Q + L.t) * WP + (mt0 + u * mstep) * 8 + L.g];
#pragma unroll
  for (int i = 0; i < NPA; ++i) {
    const int la = pa_la(i), rb = pa_rb(i);
    const int ia0 = la + rb - P, ia1 = ia0 + 1;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      double z0 = 0.0, z1 = 0.0;
      double& r0 = (ia0 >= 0 && ia0 < TA) ? acc[u][clampi(ia0, 0, TA - 1)][rb] : z0;
      double& r1 = (ia1 >= 0 && ia1 < TA) ? acc[u][clampi(ia1, 0, TA - 1)][rb + 1] : z1;
      dmma(r0, r1, av[u][la], ba[i], r0, r1);
    }
  }
  const int t = L.t;
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    const int col = (mt0 + u * mstep) * 8 + L.g;
#pragma unroll
    for (int ia = 0; ia < TA; ++ia) {
      double hi, lo;
      split_groups(acc[u][ia], t, hi, lo);
      X[(ty * NA0 + ia * NB + P + t) * XP + col] = hi;
      if (t > 0) X[(ty * NA0 + ia * NB + t - 1) * XP + col] = lo;
    }
  }
}

// ---------------------------------------------------------------- stage B
// A half unit (m-tile mt, destinations ib in {2h, 2h+1}) sees the window elements
// lb = 2h .. 2h+4 with the same pairing as stage A: fragment i of half h pairs
// r = rb, rb+1 of element lb (5 DMMAs per product instead of 10 for a full unit, so
// the 14 half units balance over the B warps).
constexpr int NPB = 10;
__host__ __device__ constexpr int pb_lb(int i) { return i < 5 ? i : i - 5 + 2; }
__host__ __device__ constexpr int pb_rb(int i) { return pa_rb(i % 5); }

// bv/bd are the warp's constant B fragments (VV and DD pair products of the axis-1
// window).  Pass 1 issues the independent X_D VV -> Y_A and X_V VV -> Y_B products,
// pass 2 adds X_V DD -> Y_A.
__device__ __forceinline__ void stage_b_half(const Lane& L, const double* X, const double (&bv)[NPB],
                                             const double (&bd)[NPB], double* Y, int mt, int h) {
  const int row = mt * 8 + L.g, a0 = row >> 2, k2 = row & 3, t = L.t;
  double yA[2][4], yB[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) yA[i][k] = yB[i][k] = 0.0;
  auto body = [&](auto hc) {
    constexpr int H = decltype(hc)::value;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1 && !L.stiff) break;
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        const int i = 5 * H + j;
        const int lb = pb_lb(i), rb = pb_rb(i);
        const int i0 = lb + rb - P - 2 * H, i1 = i0 + 1;  // local destinations (0 or 1)
        const bool v0 = i0 >= 0 && i0 < 2, v1 = i1 >= 0 && i1 < 2;
        double z0 = 0.0, z1 = 0.0, z2 = 0.0, z3 = 0.0;
        double& a0r = v0 ? yA[clampi(i0, 0, 1)][rb] : z0;
        double& a1r = v1 ? yA[clampi(i1, 0, 1)][rb + 1] : z1;
        double& b0r = v0 ? yB[clampi(i0, 0, 1)][rb] : z2;
        double& b1r = v1 ? yB[clampi(i1, 0, 1)][rb + 1] : z3;
        const int xo = (lb * Q + t) * Q + k2;
        const double xv = X[(0 * NA0 + a0) * XP + xo];
        if (pass == 0) {
          if (L.stiff) {
            const double xd = X[(1 * NA0 + a0) * XP + xo];
            dmma(a0r, a1r, xd, bv[i], a0r, a1r);
            dmma(b0r, b1r, xv, bv[i], b0r, b1r);
          } else {
            dmma(a0r, a1r, xv, bv[i], a0r, a1r);
          }
        } else {
          dmma(a0r, a1r, xv, bd[i], a0r, a1r);
        }
      }
    }
  };
  if (h == 0) body(std::integral_constant<int, 0>());
  else body(std::integral_constant<int, 1>());
#pragma unroll
  for (int il = 0; il < 2; ++il) {
    const int ib = 2 * h + il;
    double hA, lA, hB, lB;
    split_groups(yA[il], t, hA, lA);
    split_groups(yB[il], t, hB, lB);
    const int ch = (a0 * TB + ib) * NB + P + t;
    Y[(0 * Q + k2) * YP + ch] = hA;
    if (L.stiff) Y[(1 * Q + k2) * YP + ch] = hB;
    if (t > 0) {
      const int cl = (a0 * TB + ib) * NB + t - 1;
      Y[(0 * Q + k2) * YP + cl] = lA;
      if (L.stiff) Y[(1 * Q + k2) * YP + cl] = lB;
    }
  }
}

// ---------------------------------------------------------------- stage S
// NM m-tiles mt = ws + NWS i.  The rolling-row accumulators live in shared memory,
// one private slot per (m-tile, row slot, band group, lane), and are the DMMA C
// operands: column k = 2nt + j (r = k) of element e2 belongs to row e2 + k, i.e.
// slot (PHI + k) & 3, and to band group hi (d = 3+t) if k < 4-t, else lo (d = t-1).
//
// A row's group receives its first contribution at k = 3 (lo) or k = 3-t (hi): that
// DMMA takes C = 0 instead of the slot, so slots are never re-zeroed.  Row e2 (slot
// PHI) is complete after its k = 0 product: the hi value goes from the register
// straight to the CSR row and the lo value (complete since the previous element) is
// read once from its slot -- the row flush is fused into the stage.
__device__ __forceinline__ int rs_idx(int mt, int slot, int grp, int lane) {
  return ((mt * 4 + slot) * 2 + grp) * 32 + lane;
}

// destination of row I2's values for this lane: hi at band offset dh, lo at dl (or -1)
struct RowDst {
  int64_t pre2;
  int c2, dh, dl;
};

// {band_prefix(I2), band_cnt(I2)}: from the shared table when it holds the mesh's rows
__device__ __forceinline__ int2 band_of(const double* sm, int I2, int64_t N) {
  if (P3_BT && N <= NBT) return reinterpret_cast<const int2*>(sm + OFF_BT)[I2];
  return make_int2((int)band_prefix(I2, P, N), (int)band_cnt(I2, P, N));
}

__device__ __forceinline__ RowDst row_dst(int t, int I2, int64_t N, const double* sm) {
  RowDst r;
  const int lod2 = max(0, P - I2);
  const int2 b = band_of(sm, I2, N);
  r.c2 = b.y;
  r.pre2 = b.x;
  r.dh = P + t - lod2;
  r.dl = t - 1 - lod2;
  if (r.dh >= r.c2) r.dh = -1;
  if (t == 0 || r.dl >= r.c2) r.dl = -1;
  return r;
}

__device__ __forceinline__ void store_pair(const GsfArgs& a, int m, const int64_t* pb, const int* pc,
                                           const RowDst& rd, double hi, double lo) {
  if (m >= 0) {
    const int rc = m >> 16, b01 = m & 0xffff;
    double* row = a.values + pb[rc] + (int64_t)pc[rc] * rd.pre2 + b01 * rd.c2;
    if (rd.dh >= 0) row[rd.dh] = hi;
    if (rd.dl >= 0) row[rd.dl] = lo;
  }
}

template <int PHI, int I0, int NM>
__device__ __forceinline__ void stage_s_batch(const Lane& L, int ws, const double* Y, double* Rs,
                                              const double (&b0)[2], const double (&b1)[2],
                                              const int (&meta)[MT_S_PER_WARP], const int64_t* pb,
                                              const int* pc, const GsfArgs& a, const RowDst& rd) {
  const int g = L.g, t = L.t;
  double a0[NM], a1[NM], cc[NM][2][2], lo[NM];
  int p[NM][2][2];
  if (MT_S % NWS != 0 && ws + (I0 + NM - 1) * NWS >= MT_S) {
    // uneven split: the last m-tile of this batch does not exist for this warp
    if constexpr (NM > 1) stage_s_batch<PHI, I0, NM - 1>(L, ws, Y, Rs, b0, b1, meta, pb, pc, a, rd);
    return;
  }
#pragma unroll
  for (int i = 0; i < NM; ++i) {
    const int mt = ws + (I0 + i) * NWS;
    a0[i] = Y[(0 * Q + t) * YP + mt * 8 + g];
    a1[i] = L.stiff ? Y[(1 * Q + t) * YP + mt * 8 + g] : 0.0;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int k = 2 * nt + j;
        p[i][nt][j] = rs_idx(mt, (PHI + k) & 3, k < 4 - t ? 0 : 1, L.lane);
        cc[i][nt][j] = (k == 3 || k == 3 - t) ? 0.0 : Rs[p[i][nt][j]];
      }
    lo[i] = Rs[rs_idx(mt, PHI, 1, L.lane)];
  }
#pragma unroll
  for (int i = 0; i < NM; ++i)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
      dmma(cc[i][nt][0], cc[i][nt][1], a0[i], b0[nt], cc[i][nt][0], cc[i][nt][1]);
  if (L.stiff) {
#pragma unroll
    for (int i = 0; i < NM; ++i)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
        dmma(cc[i][nt][0], cc[i][nt][1], a1[i], b1[nt], cc[i][nt][0], cc[i][nt][1]);
  }
#pragma unroll
  for (int i = 0; i < NM; ++i) {
#pragma unroll
    for (int k = 1; k < 4; ++k) Rs[p[i][k >> 1][k & 1]] = cc[i][k >> 1][k & 1];
#ifndef P3_ABL_NOSTORE
    store_pair(a, meta[I0 + i], pb, pc, rd, cc[i][0][0], lo[i]);
#else
    if (cc[i][0][0] == 1.2345e-300) store_pair(a, meta[I0 + i], pb, pc, rd, cc[i][0][0], lo[i]);
#endif
  }
}

// axis-2 B fragments of element e2 (value and derivative pair products), for the first
// element; later elements go through s_raw_load / s_raw_form below
// (FOLD: the axis weights live in the fragments -- ws = w_k2 h_e2 / 2 times the Jacobian
// here -- and W is the raw coefficient; the same arithmetic as k_gsf3_p3s<FOLD>, so slab rows
// stay bitwise equal to the whole-mesh rows)
template <bool FOLD>
__device__ __forceinline__ void s_fragments(const Lane& L, const GsfArgs& a, int e2, double ws, double (&b0)[2],
                                            double (&b1)[2]) {
  const int g = L.g, t = L.t;
  const double* V2 = a.V + (int64_t)e2 * M * Q;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int r = bcol_r(nt, g), s = bcol_s(nt, g);
    // (FOLD: explicit roundings, so k_gsf3_p3 and k_gsf3_p3s form bitwise equal fragments
    // whatever the compiler contracts)
    const double vv = FOLD ? __dmul_rn(__ldg(V2 + r * Q + t), __ldg(V2 + s * Q + t))
                           : __ldg(V2 + r * Q + t) * __ldg(V2 + s * Q + t);
    b0[nt] = FOLD ? __dmul_rn(vv, ws) : vv;
    b1[nt] = 0.0;
    if (L.stiff) {
      const double* D2 = a.D + (int64_t)e2 * M * Q;
      if (FOLD) {
        double z = __dmul_rn(__ldg(D2 + r * Q + t), __ldg(D2 + s * Q + t));
        if (L.smass) z = __dadd_rn(z, vv);
        b1[nt] = __dmul_rn(z, ws);
      } else {
        double z = __ldg(D2 + r * Q + t) * __ldg(D2 + s * Q + t);
        if (L.smass) z += vv;
        b1[nt] = z;
      }
    }
  }
}

// the same in two halves: the raw table values of element e2 are loaded at the end of
// column e2-1 and their products formed at the start of column e2, so the global-load
// latency is not waited on where it is issued (0.5223 -> 0.5205 ms on C3)
struct SRaw {
  double v[2][2], d[2][2], ws;
};
template <bool FOLD>
__device__ __forceinline__ void s_raw_load(const Lane& L, const GsfArgs& a, int e2, double ws, SRaw& w) {
  const int g = L.g, t = L.t;
  const double* V2 = a.V + (int64_t)e2 * M * Q;
  const double* D2 = a.D + (int64_t)e2 * M * Q;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int r = bcol_r(nt, g), s = bcol_s(nt, g);
    w.v[nt][0] = __ldg(V2 + r * Q + t);
    w.v[nt][1] = __ldg(V2 + s * Q + t);
    w.d[nt][0] = w.d[nt][1] = 0.0;
    if (L.stiff) {
      w.d[nt][0] = __ldg(D2 + r * Q + t);
      w.d[nt][1] = __ldg(D2 + s * Q + t);
    }
  }
  if (FOLD) w.ws = ws;
}
template <bool FOLD>
__device__ __forceinline__ void s_raw_form(const Lane& L, const SRaw& w, double (&b0)[2], double (&b1)[2]) {
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const double vv = FOLD ? __dmul_rn(w.v[nt][0], w.v[nt][1]) : w.v[nt][0] * w.v[nt][1];
    b0[nt] = FOLD ? __dmul_rn(vv, w.ws) : vv;
    b1[nt] = 0.0;
    if (L.stiff) {
      if (FOLD) {
        double z = __dmul_rn(w.d[nt][0], w.d[nt][1]);
        if (L.smass) z = __dadd_rn(z, vv);
        b1[nt] = __dmul_rn(z, w.ws);
      } else {
        double z = w.d[nt][0] * w.d[nt][1];
        if (L.smass) z += vv;
        b1[nt] = z;
      }
    }
  }
}

template <int PHI>
__device__ __forceinline__ void stage_s(const Lane& L, int ws, const double* Y, double* Rs,
                                        const GsfArgs& a, int e2, const int (&meta)[MT_S_PER_WARP],
                                        const int64_t* pb, const int* pc, int64_t N,
                                        const double (&b0)[2], const double (&b1)[2]) {
  const int t = L.t;
  const RowDst rd = row_dst(t, e2, N, Rs - OFF_R);  // Rs = sm + OFF_R
  // batches of at most 4 m-tiles (loads of a batch issued before its DMMAs)
  constexpr int B0 = MT_S_PER_WARP <= 4 ? MT_S_PER_WARP : (MT_S_PER_WARP <= 8 ? (MT_S_PER_WARP + 1) / 2 : 4);
  constexpr int R1 = MT_S_PER_WARP - B0;
  constexpr int B1 = R1 <= 4 ? R1 : (R1 + 1) / 2;
  constexpr int B2 = R1 - B1;
  static_assert(B2 <= 4, "stage S batches");
  stage_s_batch<PHI, 0, B0>(L, ws, Y, Rs, b0, b1, meta, pb, pc, a, rd);
  if constexpr (B1 > 0) stage_s_batch<PHI, B0, B1>(L, ws, Y, Rs, b0, b1, meta, pb, pc, a, rd);
  if constexpr (B2 > 0) stage_s_batch<PHI, B0 + B1, B2>(L, ws, Y, Rs, b0, b1, meta, pb, pc, a, rd);
}

// Rows K .. K+P-1 (no element e2 = I2): both groups are complete in their slots.
__device__ __forceinline__ void flush_tail(const Lane& L, int ws, const double* Rs, int I2,
                                           const int (&meta)[MT_S_PER_WARP], const int64_t* pb,
                                           const int* pc, const GsfArgs& a, int64_t N) {
  const RowDst rd = row_dst(L.t, I2, N, Rs - OFF_R);
  const int sl = I2 & 3;
#pragma unroll
  for (int i = 0; i < MT_S_PER_WARP; ++i) {
    const int mt = ws + i * NWS;
    if (mt < MT_S)
      store_pair(a, meta[i], pb, pc, rd, Rs[rs_idx(mt, sl, 0, L.lane)], Rs[rs_idx(mt, sl, 1, L.lane)]);
  }
}

// W[(la,k0)][(g1,k2)] = c w0 w1 w2 jac on the CTA's quadrature slab of column e2
__device__ __forceinline__ void form_w(double* W, const double* wq, const GsfArgs& a, int e2,
                                       int i00, int i10, int e0lo, int e0hi, int tid, int nt, bool raw = false) {
  const int K = a.K;
  for (int u = tid; u < LA * Q * NCOL; u += nt) {
    const int row = u / NCOL, col = u - row * NCOL;
    const int la = row >> 2, k0 = row & 3;
    const int g1 = col >> 2, k2 = col & 3, lb = g1 >> 2, k1 = g1 & 3;
    const int e0 = i00 - P + la, e1 = i10 - P + lb;
    double w = 0.0;
    if (e0 >= e0lo && e0 < e0hi && e1 >= 0 && e1 < K) {
      const double cf = a.coef ? __ldg(a.coef + (((int64_t)e0 * K + e1) * K + e2) * (Q * Q * Q) +
                                       (k0 * Q + k1) * Q + k2)
                               : a.coef_scalar;
      w = raw ? cf
              : axis_w(wq, a.wt, e0, k0, Q) * axis_w(wq, a.wt, e1, k1, Q) * axis_w(wq, a.wt, e2, k2, Q) *
                    a.jac * cf;
    }
    W[row * WP + col] = w;
  }
}

// The coefficient field of element column e2 over the tile's window, copied asynchronously into
// W (FOLD: W is the raw coefficient).  For fixed (la, k0, lb) the 16 values (k1, k2) are
// contiguous in memory and in the W row; out-of-mesh / out-of-slab elements are zero-filled.
__device__ __forceinline__ void copy_coef_column(double* W, const GsfArgs& a, int e2, int i00, int i10, int e0lo,
                                                 int e0hi, int tid, int nt) {
  const int K = a.K;
  const bool al16 = (reinterpret_cast<uintptr_t>(a.coef) & 15) == 0;  // else 8-byte word copies
  const int np = al16 ? 8 : 16, wd = al16 ? 2 : 1;
  for (int u = tid; u < LA * Q * LB * np; u += nt) {
    const int part = u % np, seg = u / np, row = seg / LB, lb = seg - row * LB;
    const int la = row >> 2, k0 = row & 3;
    const int e0 = i00 - P + la, e1 = i10 - P + lb;
    const bool ok = e0 >= e0lo && e0 < e0hi && e1 >= 0 && e1 < K;
    const double* src = ok ? a.coef + (((int64_t)e0 * K + e1) * K + e2) * (Q * Q * Q) + k0 * (Q * Q) + part * wd : a.coef;
    const unsigned dst = (unsigned)__cvta_generic_to_shared(W + row * WP + lb * (Q * Q) + part * wd);
    if (al16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

#ifdef IGA_PHASE_TIMING
// tools/gsf_phase.cu: per-warp clock64 at the end of each role's work, iterations 8..11
__device__ long long g_phase[4][NT / 32][3];
#define PT(idx)                                                                           \
  if (blockIdx.x == IGA_PHASE_TIMING && L.lane == 0 && it >= 8 && it < 12)                \
    g_phase[it - 8][warp][idx] = clock64();
#else
#define PT(idx)
#endif

template <bool FOLD>
__global__ void __launch_bounds__(NT, 1) k_gsf3_p3(GsfArgs a) {
  extern __shared__ double sm[];
  const int tid = threadIdx.x, warp = tid >> 5;
  Lane L;
  L.lane = tid & 31; L.g = L.lane >> 2; L.t = L.lane & 3;
  L.stiff = a.op != IGA_OP_MASS;
  L.smass = a.op == IGA_OP_STIFFNESS_MASS;
  double* W = sm + OFF_W;
  double* BA = sm + OFF_BA;
  double* BB = sm + OFF_BB;
  double* wq = sm + OFF_WQ;
  int64_t* pb = reinterpret_cast<int64_t*>(sm + OFF_PB);
  int* pc = reinterpret_cast<int*>(sm + OFF_PC);
  const int K = a.K;
  const int64_t N = (int64_t)K + P;
  const int tile0 = blockIdx.x / a.tiles1, tile1 = blockIdx.x % a.tiles1;
  const int i00 = a.plane_begin + tile0 * TA, i10 = tile1 * TB;
  const int e0lo = max(a.el_begin, 0), e0hi = min(a.el_end, K);

  // ---- constant B fragments of axes 0 and 1 (pair products of the window elements)
  for (int u = tid; u < 2 * LA * 32; u += NT) {
    const int ln = u & 31, la = (u >> 5) % LA, type = u / (32 * LA);
    const int gg = ln >> 2, tt = ln & 3, e0 = i00 - P + la;
    const int r = pa_rb(la) + (gg & 1), sc = (r + (gg >> 1)) & 3;
    double v = 0.0;
    if (e0 >= 0 && e0 < K && (type == 0 || L.stiff)) {
      const double* T = (type == 0 ? a.V : a.D) + (int64_t)e0 * M * Q;
      v = T[r * Q + tt] * T[sc * Q + tt];
      if (FOLD) v = __dmul_rn(v, axis_w(a.weights, a.wt, e0, tt, Q));
    }
    BA[u] = v;
  }
  for (int u = tid; u < 2 * NPB * 32; u += NT) {
    const int ln = u & 31, i = (u >> 5) % NPB, prod = u / (32 * NPB);
    const int gg = ln >> 2, tt = ln & 3, e1 = i10 - P + pb_lb(i);
    const int r = pb_rb(i) + (gg & 1), sc = (r + (gg >> 1)) & 3;
    double v = 0.0;
    if (e1 >= 0 && e1 < K && (prod == 0 || L.stiff)) {
      const double* T = (prod == 0 ? a.V : a.D) + (int64_t)e1 * M * Q;
      v = T[r * Q + tt] * T[sc * Q + tt];
      if (FOLD) v = __dmul_rn(v, axis_w(a.weights, a.wt, e1, tt, Q));
    }
    BB[u] = v;
  }
  uint64_t* mb = reinterpret_cast<uint64_t*>(sm + OFF_MB);
  uint64_t *xfull = mb, *xempty = mb + 2, *yfull = mb + 4, *yempty = mb + 6;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(xfull + b, NWA * 32);
      mbar_init(xempty + b, NWB * 32);
      mbar_init(yfull + b, NWB * 32);
      mbar_init(yempty + b, NWS * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < Q) wq[tid] = a.weights[tid];
  if (P3_BT && N <= NBT) {
    int2* bt = reinterpret_cast<int2*>(sm + OFF_BT);
    for (int I = tid; I < N; I += NT) bt[I] = make_int2((int)band_prefix(I, P, N), (int)band_cnt(I, P, N));
  }
  if (tid < NPEN) {
    const int64_t I0 = i00 + tid / TB, I1 = i10 + tid % TB;
    pb[tid] = (I0 < N && I1 < N) ? rowptr3(I0, I1, 0, P, N) - a.base : 0;
    pc[tid] = (I0 < N && I1 < N) ? (int)(band_cnt(I0, P, N) * band_cnt(I1, P, N)) : 0;
  }
  __syncthreads();
  // Scalar coefficient on the uniform mesh: W = c w0 w1 w2 jac, formed once.  FOLD (a
  // coefficient field): the weights are in the fragments and W is the raw coefficient,
  // copied per element column with cp.async after the A warps are done with the previous
  // one (iga_gsf_p3s.cu has the double-buffered version).
  // (FOLD is the launcher's choice for a coefficient field; a general knot vector with a scalar
  // coefficient keeps the unfolded kernel and forms W per column)
  const bool w_per_step = FOLD || a.wt != nullptr;
  if (!w_per_step) form_w(W, wq, a, 0, i00, i10, e0lo, e0hi, tid, NT);
  __syncthreads();

  // pipeline: A on element column it, B on it-1, S on it-2, handed over by mbarriers
  if (warp < NWA) {
    // ------------------------------------------------------------ role A
    // warp wa owns type wa (values / derivatives; for the mass operator both warps
    // take value units) and keeps its B fragments in registers
    const int wa = warp;
    const int ty = L.stiff ? (wa & 1) : 0;
    double ba[NPA];
#pragma unroll
    for (int i = 0; i < NPA; ++i) ba[i] = BA[(ty * LA + pa_la(i)) * 32 + L.lane];
    const int mt0 = L.stiff ? (wa >> 1) : wa, mstep = L.stiff ? NWA / 2 : NWA;
    __syncthreads();  // every role holds its fragments before Y buffer 1 is written
    if (FOLD) copy_coef_column(W, a, 0, i00, i10, e0lo, e0hi, tid, NWA * 32);
    for (int it = 0; it < K; ++it) {
      PT(2);
      if (!FOLD && w_per_step) {
        if (it > 0) asm volatile("bar.sync 1, %0;\n" ::"n"(NWA * 32));  // W of it-1 consumed
        form_w(W, wq, a, it, i00, i10, e0lo, e0hi, tid, NWA * 32);
        asm volatile("bar.sync 1, %0;\n" ::"n"(NWA * 32));
      }
      if (FOLD) {
        if (it > 0) {  // W of it-1 consumed by every A warp: this column's copy starts
          asm volatile("bar.sync 1, %0;\n" ::"n"(NWA * 32));
          copy_coef_column(W, a, it, i00, i10, e0lo, e0hi, tid, NWA * 32);
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        asm volatile("bar.sync 1, %0;\n" ::"n"(NWA * 32));
      }
      const int b = it & 1;
      if (it >= 2) mbar_wait(xempty + b, ((it >> 1) - 1) & 1);
      PT(1);
      double* X = sm + OFF_X + b * SZ_X;
      int mt = mt0;
#ifndef P3_ABL_NOA
      for (; mt + mstep < MT_A; mt += 2 * mstep) stage_a_units<2>(L, W, ba, X, mt, mstep, ty);
      if (mt < MT_A) stage_a_units<1>(L, W, ba, X, mt, mstep, ty);
#endif
      mbar_arrive(xfull + b);
      PT(0);
    }
  } else if (warp < NWA + NWB) {
    // ------------------------------------------------------------ role B
    const int wb = warp - NWA;
    double bv[NPB], bd[NPB];
#pragma unroll
    for (int i = 0; i < NPB; ++i) {
      bv[i] = BB[(0 * NPB + i) * 32 + L.lane];
      bd[i] = BB[(1 * NPB + i) * 32 + L.lane];
    }
    __syncthreads();
    for (int e2 = 0; e2 < K; ++e2) {
      const int it = e2 + 1;
      PT(2);
      const int b = e2 & 1, n = e2 >> 1;
      mbar_wait(xfull + b, n & 1);
      if (n >= 1) mbar_wait(yempty + b, (n - 1) & 1);
      PT(1);
      const double* X = sm + OFF_X + b * SZ_X;
      double* Y = sm + OFF_Y + b * SZ_Y;
#ifndef P3_ABL_NOB
      for (int u = wb; u < NHB; u += NWB) stage_b_half(L, X, bv, bd, Y, u >> 1, u & 1);
#endif
      mbar_arrive(xempty + b);
      mbar_arrive(yfull + b);
      PT(0);
    }
  } else {
    // ------------------------------------------------------------ role S
    const int ws = warp - NWA - NWB;
    // per-lane store metadata of its m-tiles: pencil rc and the (d0,d1) block offset
    // b01 = (d0-lo0)*c1 + (d1-lo1) in the CSR row; -1 if the combo is outside
    int meta[MT_S_PER_WARP];
#pragma unroll
    for (int i = 0; i < MT_S_PER_WARP; ++i) {
      const int mt = ws + i * NWS;
      meta[i] = -1;
      if (mt < MT_S) {
        const int cb = mt * 8 + L.g;
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
    double* Rs = sm + OFF_R;
    for (int u = ws * 32 + L.lane; u < MT_S * 4 * 2 * 32; u += NWS * 32) Rs[u] = 0.0;
    double sb0[2], sb1[2];
    s_fragments<FOLD>(L, a, 0, FOLD ? __dmul_rn(axis_w(wq, a.wt, 0, L.t, Q), a.jac) : 1.0, sb0, sb1);
    SRaw sraw;
    __syncthreads();
    for (int e2 = 0; e2 < K; ++e2) {
      const int it = e2 + 2;
      PT(2);
      const int b = e2 & 1;
      mbar_wait(yfull + b, (e2 >> 1) & 1);
      PT(1);
      const double* Y = sm + OFF_Y + b * SZ_Y;
      if (e2 > 0) s_raw_form<FOLD>(L, sraw, sb0, sb1);
#ifdef P3_ABL_NOS
      if (e2 < 0)
#endif
      switch (e2 & 3) {
        case 0: stage_s<0>(L, ws, Y, Rs, a, e2, meta, pb, pc, N, sb0, sb1); break;
        case 1: stage_s<1>(L, ws, Y, Rs, a, e2, meta, pb, pc, N, sb0, sb1); break;
        case 2: stage_s<2>(L, ws, Y, Rs, a, e2, meta, pb, pc, N, sb0, sb1); break;
        default: stage_s<3>(L, ws, Y, Rs, a, e2, meta, pb, pc, N, sb0, sb1); break;
      }
      if (e2 + 1 < K) s_raw_load<FOLD>(L, a, e2 + 1, FOLD ? __dmul_rn(axis_w(wq, a.wt, e2 + 1, L.t, Q), a.jac) : 1.0, sraw);
      mbar_arrive(yempty + b);
      PT(0);
    }
    // rows K .. K+P-1 received their last contribution from element K-1
    for (int I2 = K; I2 < N; ++I2) flush_tail(L, ws, Rs, I2, meta, pb, pc, a, N);
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
  const bool fold = a.coef != nullptr;
  cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(fold ? p3::k_gsf3_p3<true> : p3::k_gsf3_p3<false>),
                                 p3::SMEM_BYTES);
  if (e != cudaSuccess) return check_cuda(e, "gsf_p3 smem attr");
  if (fold) p3::k_gsf3_p3<true><<<(unsigned)grid, p3::NT, p3::SMEM_BYTES, s>>>(a);
  else p3::k_gsf3_p3<false><<<(unsigned)grid, p3::NT, p3::SMEM_BYTES, s>>>(a);
  return check_cuda(cudaGetLastError(), "gsf_p3 launch");
}

}  // namespace iga

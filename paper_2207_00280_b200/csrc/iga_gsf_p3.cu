// Assembled sum factorization for p = 3, q = 4 (the headline configs C3/C5) on
// FP64 tensor cores (DMMA.8x8x4): every contraction is an MMA whose K = 4 is
// exactly one element's quadrature points.
//
// Same mathematics and tiling as k_gsf3 (iga_gsf.cu header): one CTA per
// TA x TB = 2 x 4 row pencils, streaming the elements e2 of the fastest axis.
//
// Symmetry.  S[I,J] = S[J,I], so only the upper band combos (d0,d1) >= (3,3)
// (25 of 49 per pencil) are contracted; every value is stored in its own row I
// and mirrored into row J (for (d0,d1) = (3,3) both entries belong to the same
// pencil and are computed directly).  Stage A then needs only the band offsets
// d0 >= 3 and stages B and S do about half the work.
//
// Lane layout.  Per element along an axis, the element-local product
// C[x][(r,s)] = sum_k A[x][k] T(r,k) T(s,k) has its (r,s) pairs on the MMA N
// axis.  The 16 pairs of p = 3 fit two 8-column n-tiles so that quad lane t
// holds the four columns (r, s = (r+t) mod 4), r = 0..3: one column per r.  The
// destination row of column (r,s) is then a compile-time function of (element,
// r), and its band offset d = s - r + 3 is one of two lane constants (hi: 3+t
// for r < 4-t, lo: t-1), so accumulation needs no shuffles or atomics and the
// summation order is fixed (bitwise reproducible).
//
//   stage A (axis 0): C[(g1,k2)][(r,s)] = sum_k0 W[la,k0][(g1,k2)] PA_la[k0][(r,s)]
//                     -> X_T[ia = la+r-3][d0 = 3+t][(g1,k2)]          (T = V, D)
//   stage B (axis 1): C[(a0,k2)][(r,s)] = sum_k1 X_T[a0][(lb,k1,k2)] PB_lb[k1][(r,s)]
//                     -> Y_A/Y_B[(a0, ib = lb+r-3, d1)][k2]   (upper combos only)
//   stage S (axis 2): C[c][(r,s)] = sum_k2 Y[c][k2] Z_e2[k2][(r,s)]
//                     -> R[c][row e2+r][d2]  (rolling over 4 rows, in shared memory)
//
// Warp specialisation (software pipeline over the element column e2): 4 warps run
// stage A on element e2 = it, 4 warps stage B on e2 = it-1 and 8 warps stage S
// (+ the row stores) on e2 = it-2, concurrently, with double-buffered X and Y and
// one CTA barrier per iteration, so the DMMA pipe of every SM sub-partition is
// fed by all three stages.  Constant B fragments of stages A and B live in
// registers; the rolling rows in shared memory are the DMMA C operands.
//
// Launch contract (iga_integrate_assemble): the rows of planes [pb, pe) are
// written completely.  Their lower-triangle entries pointing to planes pb-3 ..
// pb-1 are the mirrors of those planes' upper entries, so the launcher extends
// the computed planes down to pb-3 with own-row writes disabled there.
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
constexpr int NH = P + 1;                // upper band offsets d0 = 3..6
constexpr int NA0 = TA * NH;             // (ia, d0 >= 3) rows of X (8)
constexpr int NUP = 3 * NB + NH;         // upper (d0,d1) combos per pencil (25)
constexpr int NPEN = TA * TB;            // row pencils (I0, I1) of the tile
constexpr int NCOMBO = NPEN * NUP;       // combos (200)
constexpr int YP = NCOMBO + 4;           // Y pitch (== 12 mod 16: conflict-free A loads)
constexpr int NT = 512;                  // threads: 16 warps
constexpr int MT_A = NCOL / 8;           // 14 m-tiles of (g1,k2) columns
constexpr int MT_B = NA0 * Q / 8;        // 4 m-tiles of (a0,k2) rows
constexpr int MT_S = NCOMBO / 8;         // 25 m-tiles of combos
constexpr int NWA = 4, NWB = 4, NWS = 8; // warps per role (NWA even: fixed type per A warp)
constexpr int MT_S_PER_WARP = (MT_S + NWS - 1) / NWS;  // 4
static_assert(MT_B == NWB, "one stage-B m-tile per B warp");

// shared memory layout (doubles)
constexpr int SZ_X = 2 * NA0 * NCOL;              // one X buffer: [2 types][NA0][NCOL]
constexpr int SZ_Y = 2 * Q * YP;                  // one Y buffer: [2 accs * Q][YP]
constexpr int OFF_W = 0;                          // [LA*Q][WP]
constexpr int OFF_X = OFF_W + LA * Q * WP;        // 2 buffers
constexpr int OFF_Y = OFF_X + 2 * SZ_X;           // 2 buffers
constexpr int OFF_BA = OFF_Y + 2 * SZ_Y;          // [2 types][LA][2 nt][32]
constexpr int OFF_BB = OFF_BA + 2 * LA * 2 * 32;  // [2 prods][LB][2 nt][32]
constexpr int OFF_WQ = OFF_BB + 2 * LB * 2 * 32;  // weights [Q]
constexpr int OFF_R = OFF_WQ + Q;                 // rolling rows [MT_S][4 slots][2 groups][32]
constexpr int ROWU = NUP * NB;                    // upper part of an interior CSR row (175)
constexpr int MSLOT = 2 * P + 1;                  // mirror target rows in flight (J2 mod 7)
constexpr int OFF_OS = OFF_R + MT_S * 4 * 2 * 32; // own-row staging [NPEN][ROWU]
constexpr int OFF_MS = OFF_OS + NPEN * ROWU;      // mirror staging [NCOMBO][MSLOT][NB]
constexpr int OFF_PI = OFF_MS + NCOMBO * MSLOT * NB;  // pencil info: base, c01, bP  [NPEN][3]
constexpr int OFF_SEG = OFF_PI + NPEN * 3;        // mirror segment starts [NCOMBO], own
                                                  // row starts [NPEN], lengths [NPEN] (int)
constexpr int SMEM_DOUBLES = OFF_SEG + NCOMBO + NPEN + NPEN / 2;
static_assert(SMEM_DOUBLES * 8 <= 227 * 1024, "shared memory budget");
constexpr size_t SMEM_BYTES = SMEM_DOUBLES * sizeof(double);

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0,
                                     double c1) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
      : "=d"(d0), "=d"(d1)
      : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Is any column k in {2nt, 2nt+1} of window element l mapped to a destination
// index l + k - P inside [lo, hi)?
__host__ __device__ constexpr bool nt_useful(int l, int nt, int lo, int hi) {
  return (l + 2 * nt - P >= lo && l + 2 * nt - P < hi) ||
         (l + 2 * nt + 1 - P >= lo && l + 2 * nt + 1 - P < hi);
}
__host__ __device__ constexpr int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// B-fragment column mapping: lane (g, t) holds B[k=t][n=g]; column n of n-tile nt
// is the pair (r, s) = (2nt + (n&1), (r + (n>>1)) & 3).
__device__ __forceinline__ int bcol_r(int nt, int g) { return 2 * nt + (g & 1); }
__device__ __forceinline__ int bcol_s(int nt, int g) { return (bcol_r(nt, g) + (g >> 1)) & 3; }

// upper combo j (0..24) of a pencil -> band offsets (d0, d1)
__host__ __device__ __forceinline__ void combo_d(int j, int& d0, int& d1) {
  if (j < NH) { d0 = P; d1 = P + j; }
  else { d0 = P + 1 + (j - NH) / NB; d1 = (j - NH) % NB; }
}

struct Lane {
  int lane, g, t;
  bool stiff, smass;
};

// Lane masks m_k = [k < 4-t] as exact 0/1 doubles: fma(m, y, acc) adds y or nothing
// exactly, so the group sums need no data-dependent selects.
__device__ __forceinline__ double sum_hi(const double* y, int t) {
  const double m1 = t <= 2 ? 1.0 : 0.0, m2 = t <= 1 ? 1.0 : 0.0, m3 = t == 0 ? 1.0 : 0.0;
  return fma(m3, y[3], fma(m2, y[2], fma(m1, y[1], y[0])));
}
__device__ __forceinline__ void split_groups(const double* y, int t, double& hi, double& lo) {
  const double m1 = t <= 2 ? 1.0 : 0.0, m2 = t <= 1 ? 1.0 : 0.0, m3 = t == 0 ? 1.0 : 0.0;
  hi = fma(m3, y[3], fma(m2, y[2], fma(m1, y[1], y[0])));
  lo = fma(1.0 - m3, y[3], fma(1.0 - m2, y[2], (1.0 - m1) * y[1]));
}

// ---------------------------------------------------------------- stage A
// Valid (element la, n-tile) pairs of stage A (destination ia = la + k - P in [0, TA))
constexpr int NPA = 6;
__host__ __device__ constexpr int pa_la(int i) { return i < 1 ? 0 : (i < 2 ? 1 : (i < 4 ? 2 : (i < 5 ? 3 : 4))); }
__host__ __device__ constexpr int pa_nt(int i) { return i == 0 ? 1 : (i == 1 ? 1 : (i == 2 ? 0 : (i == 3 ? 1 : 0))); }

// NU units = m-tiles mt0 + i*mstep of (g1,k2) columns for the warp's type, interleaved
// for ILP; ba[] are the warp's constant B fragments; per-column accumulators
// acc[u][ia][k] are the DMMA C operands (each receives exactly one element's product).
// Only the upper band offsets d0 = 3+t (the hi group) are kept.
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
    const int la = pa_la(i), nt = pa_nt(i);
    const int ia0 = la + 2 * nt - P, ia1 = ia0 + 1;
#pragma unroll
    for (int u = 0; u < NU; ++u) {
      double z0 = 0.0, z1 = 0.0;
      double& r0 = (ia0 >= 0 && ia0 < TA) ? acc[u][clampi(ia0, 0, TA - 1)][2 * nt] : z0;
      double& r1 = (ia1 >= 0 && ia1 < TA) ? acc[u][clampi(ia1, 0, TA - 1)][2 * nt + 1] : z1;
      dmma(r0, r1, av[u][la], ba[i], r0, r1);
    }
  }
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    const int col = (mt0 + u * mstep) * 8 + L.g;
#pragma unroll
    for (int ia = 0; ia < TA; ++ia) X[(ty * NA0 + ia * NH + L.t) * NCOL + col] = sum_hi(acc[u][ia], L.t);
  }
}

// ---------------------------------------------------------------- stage B
// Valid (element lb, n-tile) pairs of stage B (destination ib = lb + k - P in [0, TB))
constexpr int NPB = 10;
__host__ __device__ constexpr int pb_lb(int i) { return i < 1 ? 0 : (i < 2 ? 1 : (i < 4 ? 2 : (i < 6 ? 3 : (i < 8 ? 4 : (i < 9 ? 5 : 6))))); }
__host__ __device__ constexpr int pb_nt(int i) { return (i == 0 || i == 1 || i == 3 || i == 5 || i == 7) ? 1 : 0; }

// unit = m-tile mt of (a0,k2) rows (a0 = (ia, d0 = 3+e)), all TB destinations ib;
// bv/bd are the warp's constant B fragments (VV and DD pair products of the axis-1
// window).  Pass 1 issues the independent X_D VV -> Y_A and X_V VV -> Y_B
// products, pass 2 adds X_V DD -> Y_A.  Only upper combos are stored.
__device__ __forceinline__ void stage_b_unit(const Lane& L, const double* X, const double (&bv)[NPB],
                                             const double (&bd)[NPB], double* Y, int mt) {
  const int row = mt * 8 + L.g, a0 = row >> 2, k2 = row & 3, t = L.t;
  const int ia = a0 / NH, e = a0 % NH;
  double yA[TB][4], yB[TB][4];
#pragma unroll
  for (int i = 0; i < TB; ++i)
#pragma unroll
    for (int k = 0; k < 4; ++k) yA[i][k] = yB[i][k] = 0.0;
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1 && !L.stiff) break;
#pragma unroll
    for (int i = 0; i < NPB; ++i) {
      const int lb = pb_lb(i), nt = pb_nt(i);
      const int i0 = lb + 2 * nt - P, i1 = i0 + 1;
      const bool v0 = i0 >= 0 && i0 < TB, v1 = i1 >= 0 && i1 < TB;
      double z0 = 0.0, z1 = 0.0, z2 = 0.0, z3 = 0.0;
      double& a0r = v0 ? yA[clampi(i0, 0, TB - 1)][2 * nt] : z0;
      double& a1r = v1 ? yA[clampi(i1, 0, TB - 1)][2 * nt + 1] : z1;
      double& b0r = v0 ? yB[clampi(i0, 0, TB - 1)][2 * nt] : z2;
      double& b1r = v1 ? yB[clampi(i1, 0, TB - 1)][2 * nt + 1] : z3;
      const int xo = (lb * Q + t) * Q + k2;
      const double xv = X[(0 * NA0 + a0) * NCOL + xo];
      if (pass == 0) {
        if (L.stiff) {
          const double xd = X[(1 * NA0 + a0) * NCOL + xo];
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
#pragma unroll
  for (int ib = 0; ib < TB; ++ib) {
    const int cb = (ia * TB + ib) * NUP;
    if (e == 0) {  // d0 = 3: upper only for d1 >= 3, i.e. the hi group (d1 = 3+t)
      const double hA = sum_hi(yA[ib], t);
      Y[(0 * Q + k2) * YP + cb + t] = hA;
      if (L.stiff) Y[(1 * Q + k2) * YP + cb + t] = sum_hi(yB[ib], t);
    } else {
      double hA, lA, hB, lB;
      split_groups(yA[ib], t, hA, lA);
      const int jh = NH + (e - 1) * NB + P + t, jl = NH + (e - 1) * NB + t - 1;
      Y[(0 * Q + k2) * YP + cb + jh] = hA;
      if (t > 0) Y[(0 * Q + k2) * YP + cb + jl] = lA;
      if (L.stiff) {
        split_groups(yB[ib], t, hB, lB);
        Y[(1 * Q + k2) * YP + cb + jh] = hB;
        if (t > 0) Y[(1 * Q + k2) * YP + cb + jl] = lB;
      }
    }
  }
}

// ---------------------------------------------------------------- stage S
// NM m-tiles mt = ws + NWS i.  The rolling-row accumulators live in shared memory,
// one private slot per (m-tile, row slot, band group, lane), and are the DMMA C
// operands: column k = 2nt + j (r = k) of element e2 belongs to row e2 + k, i.e.
// slot (PHI + k) & 3, and to band group hi (d2 = 3+t) if k < 4-t, else lo (d2 = t-1).
__device__ __forceinline__ int rs_idx(int mt, int slot, int grp, int lane) {
  return ((mt * 4 + slot) * 2 + grp) * 32 + lane;
}

template <int PHI, int I0, int NM>
__device__ __forceinline__ void stage_s_batch(const Lane& L, int ws, const double* Y, double* Rs,
                                              const double (&b0)[2], const double (&b1)[2]) {
  const int g = L.g, t = L.t;
  double a0[NM], a1[NM], cc[NM][2][2];
  int p[NM][2][2];
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
        cc[i][nt][j] = Rs[p[i][nt][j]];
      }
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
  for (int i = 0; i < NM; ++i)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int j = 0; j < 2; ++j) Rs[p[i][nt][j]] = cc[i][nt][j];
}

template <int PHI>
__device__ __forceinline__ void stage_s(const Lane& L, int ws, const double* Y, double* Rs,
                                        const GsfArgs& a, int e2) {
  const int g = L.g, t = L.t;
  const double* V2 = a.V + (int64_t)e2 * M * Q;
  double b0[2], b1[2];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int r = bcol_r(nt, g), s = bcol_s(nt, g);
    b0[nt] = __ldg(V2 + r * Q + t) * __ldg(V2 + s * Q + t);
    b1[nt] = 0.0;
    if (L.stiff) {
      const double* D2 = a.D + (int64_t)e2 * M * Q;
      double z = __ldg(D2 + r * Q + t) * __ldg(D2 + s * Q + t);
      if (L.smass) z += b0[nt];
      b1[nt] = z;
    }
  }
  static_assert(MT_S == (MT_S_PER_WARP - 1) * NWS + 1, "stage S warp split");
  stage_s_batch<PHI, 0, 3>(L, ws, Y, Rs, b0, b1);
  if (ws == 0) stage_s_batch<PHI, 3, 1>(L, ws, Y, Rs, b0, b1);
}

// Per-lane store targets of one stage-S m-tile: own row (I0, I1, .) and mirror row
// (J0, J1, .) as "row pointer of plane-pencil + c01 * prefix(I2) + b01 * c2 + d".
struct Target {
  int64_t own_base, mir_base;  // rowptr(.,.,0) - launch base
  int own_c01, mir_c01;        // c(0) * c(1) of the pencil
  int own_b01, mir_b01;        // (d0', d1') block offset inside the row (per unit c2)
  int d0, d1;                  // band offsets of the combo (own row)
  int own_s, own_rel;          // own staging row start (pen * ROWU) and block rel. to bP
  int mir_s;                   // mirror staging start (c * MSLOT * NB)
  bool own_ok, mir_ok, self;   // own row written / mirror row written / (d0,d1) == (3,3)
};

__device__ __forceinline__ void make_target(Target& tg, int c, int i00, int i10, const GsfArgs& a,
                                            int64_t N) {
  const int pen = c / NUP, j = c % NUP;
  const int ia = pen / TB, ib = pen % TB;
  int d0, d1;
  combo_d(j, d0, d1);
  tg.d0 = d0; tg.d1 = d1;
  tg.self = (d0 == P && d1 == P);
  const int64_t I0 = i00 + ia, I1 = i10 + ib;
  const int64_t J0 = I0 + d0 - P, J1 = I1 + d1 - P;
  const bool inside = I0 < N && I1 < N && J0 >= 0 && J0 < N && J1 >= 0 && J1 < N;
  tg.own_ok = inside && I0 >= a.own_begin && I0 < a.plane_end;
  tg.mir_ok = inside && !tg.self && J0 >= a.own_begin && J0 < a.mirror_end;
  tg.own_base = tg.mir_base = 0;
  tg.own_c01 = tg.mir_c01 = tg.own_b01 = tg.mir_b01 = 0;
  tg.own_s = pen * ROWU;
  tg.mir_s = c * MSLOT * NB;
  tg.own_rel = 0;
  if (tg.own_ok) {
    const int c1 = (int)band_cnt(I1, P, N);
    const int lod0 = (int)max((int64_t)0, P - I0), lod1 = (int)max((int64_t)0, P - I1);
    tg.own_base = rowptr3(I0, I1, 0, P, N) - a.base;
    tg.own_c01 = (int)(band_cnt(I0, P, N) * c1);
    tg.own_b01 = (d0 - lod0) * c1 + (d1 - lod1);
    tg.own_rel = tg.own_b01 - ((P - lod0) * c1 + (P - lod1));
  }
  if (tg.mir_ok) {
    const int c1 = (int)band_cnt(J1, P, N);
    tg.mir_base = rowptr3(J0, J1, 0, P, N) - a.base;
    tg.mir_c01 = (int)(band_cnt(J0, P, N) * c1);
    tg.mir_b01 = (2 * P - d0 - (int)max((int64_t)0, P - J0)) * c1 +
                 (2 * P - d1 - (int)max((int64_t)0, P - J1));
  }
}

// Row I2 (slot sl) is complete: each lane stages its two values (band offsets
// d2 = 3+t and t-1) per m-tile in the own-row staging (upper part of row I2) and
// in the mirror staging of target row J2 = I2 + d2 - 3 (slot J2 mod 7, position
// 2P - d2), then clears the rolling slot.
__device__ __forceinline__ void stage_rows(const Lane& L, int ws, double* Rs, int sl,
                                           const Target (&tg)[MT_S_PER_WARP], double* OS,
                                           double* MS, int I2, int64_t N) {
  const int t = L.t;
  const int c_i = (int)band_cnt(I2, P, N), lod_i = max(0, P - I2);
  const int d2v[2] = {P + t, t - 1};
  // per band offset: validity of column J2 = I2 + d2 - 3, own position, mirror slot
  bool okh[2];
  int op[2], mp[2];
  const int i2m = I2 % MSLOT;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int d2 = d2v[h];
    const int J2 = I2 + d2 - P;
    okh[h] = !(h == 1 && t == 0) && J2 >= 0 && J2 < N;
    op[h] = d2 - lod_i;
    int slot = i2m + d2 - P;
    slot = slot < 0 ? slot + MSLOT : (slot >= MSLOT ? slot - MSLOT : slot);
    mp[h] = slot * NB + (2 * P - d2);
  }
#pragma unroll
  for (int i = 0; i < MT_S_PER_WARP; ++i) {
    const int mt = ws + i * NWS;
    if (mt < MT_S) {
      const int ph = rs_idx(mt, sl, 0, L.lane), pl = rs_idx(mt, sl, 1, L.lane);
      const double v[2] = {Rs[ph], Rs[pl]};
      const Target& g = tg[i];
      const int ob = g.own_s + g.own_rel * c_i;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (!okh[h]) continue;
        if (g.own_ok) OS[ob + op[h]] = v[h];
        if (g.mir_ok) MS[g.mir_s + mp[h]] = v[h];
      }
      Rs[ph] = 0.0;
      Rs[pl] = 0.0;
    }
  }
}

// Write-out bases of the rows finished at this step: own row I2 of every pencil
// (OB[pen] = first upper position or -1, OL[pen] = upper length) and the mirror
// segment of every combo in target row J2 = I2 - 3 (SEGB[c] or -1).  Computed by
// the S lanes right after staging, read by the flat write loop after the barrier.
__device__ __forceinline__ void write_bases(const Target (&tg)[MT_S_PER_WARP], const int64_t* PI,
                                            int64_t* OB, int* OL, int64_t* SEGB, const GsfArgs& a,
                                            int I2, int64_t N, int ws, const Lane& L, int stid) {
  if (stid < NPEN) {
    const int64_t c01 = PI[stid * 3 + 1];
    const int64_t bP = PI[stid * 3 + 2];
    const int64_t c2 = band_cnt(I2, P, N);
    OB[stid] = c01 > 0 ? PI[stid * 3] + c01 * band_prefix(I2, P, N) + bP * c2 : -1;
    OL[stid] = c01 > 0 ? (int)((c01 - bP) * c2) : 0;
  }
  const int J2 = I2 - P;
  if (J2 >= 0 && L.t == 0) {
    const int64_t pre = band_prefix(J2, P, N);
    const int64_t c2 = band_cnt(J2, P, N);
#pragma unroll
    for (int i = 0; i < MT_S_PER_WARP; ++i) {
      const int mt = ws + i * NWS;
      if (mt < MT_S) {
        const Target& g = tg[i];
        SEGB[mt * 8 + L.g] = g.mir_ok ? g.mir_base + (int64_t)g.mir_c01 * pre + (int64_t)g.mir_b01 * c2 : -1;
      }
    }
  }
}

// Flat write loop: the staged upper parts of the tile's rows I2 (own) and the
// mirrored segments of target row J2 = I2 - 3; fully unrolled so every thread keeps
// its loads and stores in flight together.
__device__ __forceinline__ void write_rows(const double* OS, const double* MS, const int64_t* OB,
                                           const int* OL, const int64_t* SEGB, const GsfArgs& a,
                                           int I2, int64_t N, int stid) {
  constexpr int NOWN = NPEN * ROWU, NMIR = NCOMBO * NB, NTS = NWS * 32;
  const int J2 = I2 - P;
  const int slot = J2 >= 0 ? J2 % MSLOT : 0;
  const int c2 = J2 >= 0 ? (int)band_cnt(J2, P, N) : 0, lod = J2 >= 0 ? max(0, P - J2) : 0;
#pragma unroll
  for (int k = 0; k < (NOWN + NMIR + NTS - 1) / NTS; ++k) {
    const int u = stid + k * NTS;
    if (u < NOWN) {
      const int pen = u / ROWU, v = u - pen * ROWU;
      const int64_t ob = OB[pen];
      if (ob >= 0 && v < OL[pen]) a.values[ob + v] = OS[u];
    } else if (u < NOWN + NMIR && J2 >= 0) {
      const int w = u - NOWN, c = w / NB, d = w - c * NB;
      const int64_t sb = SEGB[c];
      if (sb >= 0 && d < c2) a.values[sb + d] = MS[(c * MSLOT + slot) * NB + lod + d];
    }
  }
}

// W[(la,k0)][(g1,k2)] = c w0 w1 w2 jac on the CTA's quadrature slab of column e2
__device__ __forceinline__ void form_w(double* W, const double* wq, const GsfArgs& a, int e2,
                                       int i00, int i10, int e0lo, int e0hi, int tid, int nt) {
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
      w = wq[k0] * wq[k1] * wq[k2] * a.jac * cf;
    }
    W[row * WP + col] = w;
  }
}

#ifdef IGA_PHASE_TIMING
// tools/gsf_phase.cu: per-warp clock64 of one CTA, iterations 8..11
__device__ long long g_phase[4][NT / 32][6];
#define PT(idx)                                                                           \
  if (blockIdx.x == IGA_PHASE_TIMING && L.lane == 0 && it >= 8 && it < 12)                \
    g_phase[it - 8][warp][idx] = clock64();
#else
#define PT(idx)
#endif

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
  const int K = a.K;
  const int64_t N = (int64_t)K + P;
  const int tile0 = blockIdx.x / a.tiles1, tile1 = blockIdx.x % a.tiles1;
  const int i00 = a.plane_begin + tile0 * TA, i10 = tile1 * TB;
  const int e0lo = max(a.el_begin, 0), e0hi = min(a.el_end, K);

  // ---- constant B fragments of axes 0 and 1 (pair products of the window elements)
  for (int u = tid; u < 2 * LA * 2 * 32; u += NT) {
    const int ln = u & 31, nt = (u >> 5) & 1, la = (u >> 6) % LA, type = u / (64 * LA);
    const int gg = ln >> 2, tt = ln & 3, e0 = i00 - P + la;
    double v = 0.0;
    if (e0 >= 0 && e0 < K && (type == 0 || L.stiff)) {
      const double* T = (type == 0 ? a.V : a.D) + (int64_t)e0 * M * Q;
      v = T[bcol_r(nt, gg) * Q + tt] * T[bcol_s(nt, gg) * Q + tt];
    }
    BA[u] = v;
  }
  for (int u = tid; u < 2 * LB * 2 * 32; u += NT) {
    const int ln = u & 31, nt = (u >> 5) & 1, lb = (u >> 6) % LB, prod = u / (64 * LB);
    const int gg = ln >> 2, tt = ln & 3, e1 = i10 - P + lb;
    double v = 0.0;
    if (e1 >= 0 && e1 < K && (prod == 0 || L.stiff)) {
      const double* T = (prod == 0 ? a.V : a.D) + (int64_t)e1 * M * Q;
      v = T[bcol_r(nt, gg) * Q + tt] * T[bcol_s(nt, gg) * Q + tt];
    }
    BB[u] = v;
  }
  if (tid < Q) wq[tid] = a.weights[tid];
  if (tid < NPEN) {
    // own-row write-out info of pencil (I0, I1): row pointer of (I0, I1, 0), c0*c1
    // (0 if the pencil's rows are not written by this launch) and the first upper block
    int64_t* PIw = reinterpret_cast<int64_t*>(sm + OFF_PI);
    const int64_t I0 = i00 + tid / TB, I1 = i10 + tid % TB;
    const bool ok = I0 < N && I1 < N && I0 >= a.own_begin && I0 < a.plane_end;
    const int64_t c1 = ok ? band_cnt(I1, P, N) : 0;
    PIw[tid * 3 + 0] = ok ? rowptr3(I0, I1, 0, P, N) - a.base : 0;
    PIw[tid * 3 + 1] = ok ? band_cnt(I0, P, N) * c1 : 0;
    PIw[tid * 3 + 2] = ok ? (P - max((int64_t)0, P - I0)) * c1 + (P - max((int64_t)0, P - I1)) : 0;
  }
  __syncthreads();
  if (a.coef == nullptr) form_w(W, wq, a, 0, i00, i10, e0lo, e0hi, tid, NT);  // step-invariant
  __syncthreads();

  const int n_it = K + 2;  // pipeline: A on it, B on it-1, S on it-2
  if (warp < NWA) {
    // ------------------------------------------------------------ role A
    // warp wa owns type wa & 1 (values / derivatives; for the mass operator all A
    // warps take value units) and keeps its B fragments in registers
    const int wa = warp;
    const int ty = L.stiff ? (wa & 1) : 0;
    double ba[NPA];
#pragma unroll
    for (int i = 0; i < NPA; ++i) ba[i] = BA[((ty * LA + pa_la(i)) * 2 + pa_nt(i)) * 32 + L.lane];
    const int mt0 = L.stiff ? (wa >> 1) : wa, mstep = L.stiff ? NWA / 2 : NWA;
    for (int it = 0; it < n_it; ++it) {
      PT(2);
      if (it < K) {
        if (a.coef != nullptr) {
          form_w(W, wq, a, it, i00, i10, e0lo, e0hi, tid, NWA * 32);
          asm volatile("bar.sync 1, %0;\n" ::"n"(NWA * 32));
        }
        double* X = sm + OFF_X + (it & 1) * SZ_X;
        int mt = mt0;
        for (; mt + mstep < MT_A; mt += 2 * mstep) stage_a_units<2>(L, W, ba, X, mt, mstep, ty);
        if (mt < MT_A) stage_a_units<1>(L, W, ba, X, mt, mstep, ty);
        PT(0);
      }
      __syncthreads();
    }
  } else if (warp < NWA + NWB) {
    // ------------------------------------------------------------ role B
    const int wb = warp - NWA;
    double bv[NPB], bd[NPB];
#pragma unroll
    for (int i = 0; i < NPB; ++i) {
      bv[i] = BB[((0 * LB + pb_lb(i)) * 2 + pb_nt(i)) * 32 + L.lane];
      bd[i] = BB[((1 * LB + pb_lb(i)) * 2 + pb_nt(i)) * 32 + L.lane];
    }
    for (int it = 0; it < n_it; ++it) {
      PT(2);
      const int e2 = it - 1;
      if (e2 >= 0 && e2 < K) {
        const double* X = sm + OFF_X + (e2 & 1) * SZ_X;
        double* Y = sm + OFF_Y + (e2 & 1) * SZ_Y;
        stage_b_unit(L, X, bv, bd, Y, wb);
        PT(0);
      }
      __syncthreads();
    }
  } else {
    // ------------------------------------------------------------ role S
    const int ws = warp - NWA - NWB;
    Target tg[MT_S_PER_WARP];
#pragma unroll
    for (int i = 0; i < MT_S_PER_WARP; ++i) {
      const int mt = ws + i * NWS;
      make_target(tg[i], mt < MT_S ? mt * 8 + L.g : 0, i00, i10, a, N);
      if (mt >= MT_S) tg[i].own_ok = tg[i].mir_ok = false;
    }
    double* Rs = sm + OFF_R;
    double* OS = sm + OFF_OS;
    double* MS = sm + OFF_MS;
    const int64_t* PI = reinterpret_cast<const int64_t*>(sm + OFF_PI);
    int64_t* SEGB = reinterpret_cast<int64_t*>(sm + OFF_SEG);
    const int stid = tid - (NWA + NWB) * 32, snt = NWS * 32;
    for (int u = stid; u < MT_S * 4 * 2 * 32; u += snt) Rs[u] = 0.0;
    int64_t* OB = SEGB + NCOMBO;
    int* OL = reinterpret_cast<int*>(OB + NPEN);
    auto finish_row = [&](int I2, int it) {
      // row I2 is complete: stage it, then write it and the mirror row I2-3
      asm volatile("bar.sync 2, %0;\n" ::"n"(NWS * 32));
      PT(3);
      stage_rows(L, ws, Rs, I2 & 3, tg, OS, MS, I2, N);
      write_bases(tg, PI, OB, OL, SEGB, a, I2, N, ws, L, stid);
      PT(4);
      asm volatile("bar.sync 2, %0;\n" ::"n"(NWS * 32));
      write_rows(OS, MS, OB, OL, SEGB, a, I2, N, stid);
      PT(5);
    };
    for (int it = 0; it < n_it; ++it) {
      PT(2);
      const int e2 = it - 2;
      if (e2 >= 0) {
        const double* Y = sm + OFF_Y + (e2 & 1) * SZ_Y;
        switch (e2 & 3) {
          case 0: stage_s<0>(L, ws, Y, Rs, a, e2); break;
          case 1: stage_s<1>(L, ws, Y, Rs, a, e2); break;
          case 2: stage_s<2>(L, ws, Y, Rs, a, e2); break;
          default: stage_s<3>(L, ws, Y, Rs, a, e2); break;
        }
        PT(0);
        finish_row(e2, it);
        PT(1);
      }
      __syncthreads();
    }
    // rows K .. K+P-1 received their last contribution from element K-1; then the
    // last P mirror rows
    for (int I2 = K; I2 < N; ++I2) finish_row(I2, 0);
    // mirror rows N-3 .. N-1: flushed as "rows" N .. N+2 whose own parts are empty
    for (int I2 = (int)N; I2 < N + P; ++I2) {
      asm volatile("bar.sync 2, %0;\n" ::"n"(NWS * 32));
      if (stid < NPEN) { OB[stid] = -1; OL[stid] = 0; }
      const int J2 = I2 - P;
      if (J2 >= 0 && L.t == 0) {
        const int64_t pre = band_prefix(J2, P, N), c2 = band_cnt(J2, P, N);
#pragma unroll
        for (int i = 0; i < MT_S_PER_WARP; ++i) {
          const int mt = ws + i * NWS;
          if (mt < MT_S)
            SEGB[mt * 8 + L.g] = tg[i].mir_ok ? tg[i].mir_base + (int64_t)tg[i].mir_c01 * pre +
                                                    (int64_t)tg[i].mir_b01 * c2 : -1;
        }
      }
      asm volatile("bar.sync 2, %0;\n" ::"n"(NWS * 32));
      write_rows(OS, MS, OB, OL, SEGB, a, I2, N, stid);
    }
  }
}

}  // namespace p3

// Rows of planes [pb, pe) are written completely: the computed planes start P
// planes earlier (own rows not written there) so that the lower-triangle entries
// pointing below pb arrive as mirrors.
int launch_gsf_p3(const GsfArgs& a0, cudaStream_t s) {
  GsfArgs a = a0;
  const int64_t N = (int64_t)a.K + p3::P;
  if (a.plane_end <= a.plane_begin) return IGA_OK;
  a.own_begin = a0.plane_begin;
  a.mirror_end = a0.plane_end;
  a.plane_begin = a0.plane_begin - p3::P > 0 ? a0.plane_begin - p3::P : 0;
  const int planes = a.plane_end - a.plane_begin;
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

// Symmetric variant of k_gsf3_p3 (iga_gsf_p3.cu): the same warp-specialised DMMA pipeline
// for p = 3, q = 4, computing only the values S[I, J] with J0 >= I0 and writing each value
// with J0 > I0 twice, at (I, J) and mirrored at (J, I) -- the matrix is symmetric
// (assembly.py:77-79 stores both triangles; SURVEY.md 9.6 allows computing one and
// mirroring at write time).
//
// Of stage A's two band groups per lane (iga_gsf_p3.cu: hi = band offset 3 + t, lo = t - 1)
// the hi group is exactly J0 >= I0, so stage A keeps only its hi sums and X has TA (p+1)
// instead of TA (2p+1) rows: stage B then runs 4 of 7 m-tiles and stage S 28 of 49 (DMMAs
// per element column 546 -> 372), and the band-group DFMAs of stage A halve.  The mirrored
// values land in another pencil's row per lane: written directly they cost 32 partial-sector
// L2 writes per warp store instruction (C3: 0.571 ms, against 0.391 without them).  Instead
// each S warp keeps per-combo rings of its mirrored values by target row (ring_put), and a
// fourth role, the emitter warps (role E, emit_all), writes every target row's values of a
// combo as one contiguous run once its last source row is done (hi runs d2' = 0..3 when
// source row J2 completes, lo runs d2' = 4..6 three columns later).  The S warps hand a row
// to the emitters through mbarriers (rfull / rfree) and may run two rows ahead of them.  With
// the S warps emitting their own runs they were the slowest role (stage B waited on their Y
// buffers: 10% of the stall samples); 20 warps cost 96 registers per thread, which the roles
// fit.  C3: 0.419 ms against 0.437 with S-warp emission and 0.509 for k_gsf3_p3.  Valid when
// the call writes every row its elements touch (sym_covers: a whole mesh, or a multi-GPU
// element slab with its interface planes); other plane ranges take k_gsf3_p3.
//
// Everything else -- tiling, the roles, the mbarrier hand-off, the rolling rows of stage S,
// the summation order of each computed value -- is k_gsf3_p3's; see its header.
#include <type_traits>

#include "iga_args.cuh"
#include "iga_dispatch.cuh"

namespace iga {
namespace p3s {

constexpr int P = 3, M = 4, Q = 4, NB = 7, NBH = P + 1;
constexpr int TA = 2, TB = 4;
constexpr int LA = TA + P, LB = TB + P;  // element windows (5, 7)
constexpr int GB = LB * Q;               // axis-1 quadrature points in the window (28)
constexpr int NCOL = GB * Q;             // (g1, k2) columns (112)
constexpr int WP = NCOL + 4;             // W row pitch (== 4 mod 16: conflict-free A loads)
constexpr int XP = NCOL + 4;             // X row pitch (== 4 mod 16: conflict-free A stores)
constexpr int NA0 = TA * NBH;            // (ia, dh) rows, d0 = P + dh >= P (8)
constexpr int NCOMBO = NA0 * TB * NB;    // (ia, dh, ib, d1) combos (224)
constexpr int YP = NCOMBO + 4;           // Y pitch (== 12 mod 16: conflict-free A loads)
constexpr int MT_A = NCOL / 8;           // 14 m-tiles of (g1,k2) columns
constexpr int MT_B = NA0 * Q / 8;        // 4 m-tiles of (a0,k2) rows
constexpr int MT_S = NCOMBO / 8;         // 28 m-tiles of combos
#ifndef P3S_NWB
#define P3S_NWB 5
#endif
#ifndef P3S_NWS
#define P3S_NWS 7
#endif
#ifndef P3S_NWA
#define P3S_NWA 4
#endif
#ifndef P3S_NWE
#define P3S_NWE 4
#endif
// warps per role (NWA even: fixed type per A warp); the NWE emitter warps write the mirrored
// runs out of the S warps' rings.  17..20 warps cost the same 96 registers per thread (5 warps
// per SM sub-partition), so the emitters come in fours.
constexpr int NWA = P3S_NWA, NWB = P3S_NWB, NWS = P3S_NWS, NWE = P3S_NWE;
static_assert(NWA % 2 == 0, "stage-A warps come in (value, derivative) pairs");
static_assert(NWE >= 1, "role E writes the mirrored runs");
constexpr int NT = 32 * (NWA + NWB + NWS + NWE);  // threads (20 warps by default: 4 A, 5 B, 7 S, 4 E)
constexpr int MT_S_PER_WARP = (MT_S + NWS - 1) / NWS;  // 4
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
// mirror metadata per ring combo c = ((ws, i), g), written by the S warps and read once by
// the emitters: CSR base of the target pencil (int64) and (c0 c1, (d0, d1) block offset) of
// the target row (int pair); block -1: no mirror
constexpr int NRC = NWS * MT_S_PER_WARP * 8;       // ring combos (224)
constexpr int OFF_MM = OFF_R + MT_S * 4 * 2 * 32;  // [NRC][2]
// axis-2 band table {band_prefix(I2), band_cnt(I2)} for meshes with N <= NBT rows (else computed)
constexpr int NBT = 512;
constexpr int OFF_BT = OFF_MM + NRC * 2;  // int2 [NBT]
constexpr int OFF_RING = OFF_BT + NBT;     // [NRC][RING]
// per ring combo: the mirrored values by target row J2 -- hi runs [J2 mod HS][d2' 0..3], lo runs
// [J2 mod 4][d2' 4..6] -- so they leave as contiguous runs.  HS = 8 hi slots let the S warps
// run two rows ahead of the emitters (LAG; ring_put / role E below).  The folded kernel
// (FOLD, coefficient fields) keeps 4 and one row, and spends the shared memory on a second
// W buffer, so the next element column's coefficients are copied while this one is used.
template <bool FOLD>
struct Rg {
  static constexpr int HS = FOLD ? 4 : 8, LAG = FOLD ? 1 : 2;
  static constexpr int LO = HS * 4, RING = LO + 12;
  static constexpr int OFF_W2 = OFF_RING + NRC * RING;  // second W buffer (FOLD)
  static constexpr int OFF_MB = FOLD ? OFF_W2 + LA * Q * WP : OFF_W2;  // mbarriers
  static constexpr int SMEM_DOUBLES = OFF_MB + 12;
  static_assert(SMEM_DOUBLES * 8 <= 227 * 1024, "shared memory budget");
  static_assert(OFF_W2 % 2 == 0, "16-byte aligned cp.async destinations");
  static constexpr size_t SMEM_BYTES = SMEM_DOUBLES * sizeof(double);
};

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
// exactly, so the group sums need no data-dependent selects (k_gsf3_p3's order: the hi
// values are bitwise those of k_gsf3_p3)
__device__ __forceinline__ void split_groups(const double* y, int t, double& hi, double& lo) {
  const double m1 = t <= 2 ? 1.0 : 0.0, m2 = t <= 1 ? 1.0 : 0.0, m3 = t == 0 ? 1.0 : 0.0;
  hi = fma(m3, y[3], fma(m2, y[2], fma(m1, y[1], y[0])));
  lo = fma(1.0 - m3, y[3], fma(1.0 - m2, y[2], (1.0 - m1) * y[1]));
}
__device__ __forceinline__ double hi_group(const double* y, int t) {
  const double m1 = t <= 2 ? 1.0 : 0.0, m2 = t <= 1 ? 1.0 : 0.0, m3 = t == 0 ? 1.0 : 0.0;
  return fma(m3, y[3], fma(m2, y[2], fma(m1, y[1], y[0])));
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
    for (int ia = 0; ia < TA; ++ia)  // only the J0 >= I0 group: row (ia, dh = t)
      X[(ty * NA0 + ia * NBH + t) * XP + col] = hi_group(acc[u][ia], t);
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

// {band_prefix(I), band_cnt(I)} of axis-2 row I: from the shared table when it holds the mesh
__device__ __forceinline__ int2 band_of(const int2* bt, int I, int64_t N) {
  if (N <= NBT) return bt[I];
  return make_int2((int)band_prefix(I, P, N), (int)band_cnt(I, P, N));
}

__device__ __forceinline__ RowDst row_dst(int t, int I2, int64_t N, const int2* bt) {
  RowDst r;
  const int lod2 = max(0, P - I2);
  const int2 b = band_of(bt, I2, N);
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

// Row I2's mirrored values into this lane group's rings: hi -> target J2 = I2 + t at d2' = 3 - t
// (slot J2 mod 8), lo -> J2 = I2 + t - 4 at d2' = 7 - t (ring entry d2' - 4, slot J2 mod 4).
// The hi slot was last read for target J2 - 8, emitted with row J2 - 8 <= I2 - 5; the lo slot
// for target J2 - 4, emitted with row J2 - 1 <= I2 - 2: row I2's values may be put once the
// emitters are done with row I2 - 2.
template <bool FOLD>
__device__ __forceinline__ void ring_put(double* rg, int i, int g, int t, int I2, double hi, double lo) {
  using G = Rg<FOLD>;
  double* r = rg + (i * 8 + g) * G::RING;
  r[((I2 + t) & (G::HS - 1)) * 4 + (3 - t)] = hi;
  if (t > 0) r[G::LO + ((I2 + t) & 3) * 3 + (3 - t)] = lo;
}

// Target row J2's complete runs, written by the emitter warps (role E): hi (d2' = t) or lo
// (d2' = 4 + t, t < 3), one contiguous run per combo (the 4 lanes of a group write consecutive
// values).  The ring combos, in ring order, are dealt to the NWE * 8 lane groups; a lane keeps
// t and the CSR metadata of its ENJ combos in registers, so a row's emission is ENJ
// independent {ring load, address, store} sequences.
constexpr int ENG = NWE * 8;                   // lane groups
constexpr int ENJ = (NRC + ENG - 1) / ENG;     // combos per lane (7)
struct EMeta {
  double* row[ENJ];  // values + CSR base of the target pencil
  int cx[ENJ], cy[ENJ];
};
template <bool HI, bool FOLD>
__device__ __forceinline__ void emit_all(const GsfArgs& a, const double* sm, const EMeta& em, int et, int J2,
                                         int64_t N) {
  const int2 b = band_of(reinterpret_cast<const int2*>(sm + OFF_BT), J2, N);
  const int t = et & 3;
  const int off = (HI ? t : 4 + t) - max(0, P - J2);
  const bool ok = (HI || t < 3) && off >= 0 && off < b.y;
  using G = Rg<FOLD>;
  const double* r = sm + OFF_RING + (et >> 2) * G::RING +
                    (HI ? (J2 & (G::HS - 1)) * 4 + t : G::LO + (J2 & 3) * 3 + (t < 3 ? t : 0));
  double v[ENJ];
#pragma unroll
  for (int j = 0; j < ENJ; ++j) v[j] = em.cy[j] >= 0 ? r[j * ENG * G::RING] : 0.0;
  // offsets within a pencil fit 32 bits: c0 c1 band_prefix(J2) + (block) band_cnt(J2) + off < 343 N
#pragma unroll
  for (int j = 0; j < ENJ; ++j)
    if (ok && em.cy[j] >= 0) em.row[j][em.cx[j] * b.x + em.cy[j] * b.y + off] = v[j];
}

template <int PHI, int I0, int NM, bool FOLD>
__device__ __forceinline__ void stage_s_batch(const Lane& L, int ws, const double* Y, double* Rs,
                                              const double (&b0)[2], const double (&b1)[2],
                                              const int (&meta)[MT_S_PER_WARP], const int64_t* pb,
                                              const int* pc, const GsfArgs& a, const RowDst& rd,
                                              double* rg, int e2) {
  const int g = L.g, t = L.t;
  double a0[NM], a1[NM], cc[NM][2][2], lo[NM];
  int p[NM][2][2];
  if (MT_S % NWS != 0 && ws + (I0 + NM - 1) * NWS >= MT_S) {
    // uneven split: the last m-tile of this batch does not exist for this warp
    if constexpr (NM > 1) stage_s_batch<PHI, I0, NM - 1, FOLD>(L, ws, Y, Rs, b0, b1, meta, pb, pc, a, rd, rg, e2);
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
  // the emitters are done with row e2 - LAG (ring_put): its slots are reused from here on
  constexpr int LAG = Rg<FOLD>::LAG;
  if (I0 == 0 && e2 >= LAG)
    mbar_wait(reinterpret_cast<uint64_t*>(Rs - OFF_R + Rg<FOLD>::OFF_MB) + 10 + ((e2 - LAG) & 1),
              ((e2 - LAG) >> 1) & 1);
#pragma unroll
  for (int i = 0; i < NM; ++i) {
#pragma unroll
    for (int k = 1; k < 4; ++k) Rs[p[i][k >> 1][k & 1]] = cc[i][k >> 1][k & 1];
    store_pair(a, meta[I0 + i], pb, pc, rd, cc[i][0][0], lo[i]);
    ring_put<FOLD>(rg, I0 + i, g, t, e2, cc[i][0][0], lo[i]);
  }
}

// axis-2 B fragments of element e2 (value and derivative pair products), for the first
// element; later elements go through s_raw_load / s_raw_form below
// (ws: the axis-2 weight w_k2 h_e2 / 2 times the Jacobian when the weights are folded into the
// fragments, else 1 -- see `folded` in the kernel)
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

// The coefficient field of element column e2 over the tile's window, copied asynchronously into
// W (folded mode: W is the raw coefficient).  For fixed (la, k0, lb) the 16 values (k1, k2) are
// contiguous in memory (128 aligned bytes) and in the W row; out-of-mesh / out-of-slab
// elements are zero-filled (source size 0).
__device__ __forceinline__ void copy_coef_column(double* W, const GsfArgs& a, int e2, int i00, int i10, int e0lo,
                                                 int e0hi, int tid, int nt) {
  const int K = a.K;
  if (reinterpret_cast<uintptr_t>(a.coef) & 15) {  // a caller's 8-byte aligned field: word copies
    for (int u = tid; u < LA * Q * LB * 16; u += nt) {
      const int part = u & 15, seg = u >> 4, row = seg / LB, lb = seg - row * LB;
      const int la = row >> 2, k0 = row & 3;
      const int e0 = i00 - P + la, e1 = i10 - P + lb;
      const bool ok = e0 >= e0lo && e0 < e0hi && e1 >= 0 && e1 < K;
      const double* src = ok ? a.coef + (((int64_t)e0 * K + e1) * K + e2) * (Q * Q * Q) + k0 * (Q * Q) + part : a.coef;
      const unsigned dst = smem_u32(W + row * WP + lb * (Q * Q) + part);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    return;
  }
  for (int u = tid; u < LA * Q * LB * 8; u += nt) {
    const int part = u & 7, seg = u >> 3, row = seg / LB, lb = seg - row * LB;
    const int la = row >> 2, k0 = row & 3;
    const int e0 = i00 - P + la, e1 = i10 - P + lb;
    const bool ok = e0 >= e0lo && e0 < e0hi && e1 >= 0 && e1 < K;
    const double* src = ok ? a.coef + (((int64_t)e0 * K + e1) * K + e2) * (Q * Q * Q) + k0 * (Q * Q) + part * 2 : a.coef;
    const unsigned dst = smem_u32(W + row * WP + lb * (Q * Q) + part * 2);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int PHI, bool FOLD>
__device__ __forceinline__ void stage_s(const Lane& L, int ws, const double* Y, double* Rs,
                                        const GsfArgs& a, int e2, const int (&meta)[MT_S_PER_WARP],
                                        const int64_t* pb, const int* pc, int64_t N,
                                        const double (&b0)[2], const double (&b1)[2], double* rg) {
  const int t = L.t;
  const int2* bt = reinterpret_cast<const int2*>(Rs - OFF_R + OFF_BT);  // Rs = sm + OFF_R
  const RowDst rd = row_dst(t, e2, N, bt);
  // batches of at most 4 m-tiles (loads of a batch issued before its DMMAs)
  constexpr int B0 = MT_S_PER_WARP <= 4 ? MT_S_PER_WARP : (MT_S_PER_WARP <= 8 ? (MT_S_PER_WARP + 1) / 2 : 4);
  constexpr int R1 = MT_S_PER_WARP - B0;
  constexpr int B1 = R1 <= 4 ? R1 : (R1 + 1) / 2;
  constexpr int B2 = R1 - B1;
  static_assert(B2 <= 4, "stage S batches");
  stage_s_batch<PHI, 0, B0, FOLD>(L, ws, Y, Rs, b0, b1, meta, pb, pc, a, rd, rg, e2);
  if constexpr (B1 > 0) stage_s_batch<PHI, B0, B1, FOLD>(L, ws, Y, Rs, b0, b1, meta, pb, pc, a, rd, rg, e2);
  if constexpr (B2 > 0) stage_s_batch<PHI, B0 + B1, B2, FOLD>(L, ws, Y, Rs, b0, b1, meta, pb, pc, a, rd, rg, e2);
}

// Rows K .. K+P-1 (no element e2 = I2): both groups are complete in their slots.
template <bool FOLD>
__device__ __forceinline__ void flush_tail(const Lane& L, int ws, const double* Rs, int I2,
                                           const int (&meta)[MT_S_PER_WARP], const int64_t* pb,
                                           const int* pc, const GsfArgs& a, int64_t N, double* rg) {
  const int2* bt = reinterpret_cast<const int2*>(Rs - OFF_R + OFF_BT);  // Rs = sm + OFF_R
  const RowDst rd = row_dst(L.t, I2, N, bt);
  const int sl = I2 & 3;
#pragma unroll
  for (int i = 0; i < MT_S_PER_WARP; ++i) {
    const int mt = ws + i * NWS;
    if (mt < MT_S) {
      const double hi = Rs[rs_idx(mt, sl, 0, L.lane)], lo = Rs[rs_idx(mt, sl, 1, L.lane)];
      store_pair(a, meta[i], pb, pc, rd, hi, lo);
      ring_put<FOLD>(rg, i, L.g, L.t, I2, hi, lo);
    }
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


// FOLD: the axis weights live in the fragments and W is the raw coefficient (see `folded`
// below); the launcher picks it for a coefficient field or a general knot vector
template <bool FOLD>
__global__ void __launch_bounds__(NT, 1) k_gsf3_p3s(GsfArgs a) {
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
  uint64_t* mb = reinterpret_cast<uint64_t*>(sm + Rg<FOLD>::OFF_MB);
  uint64_t *xfull = mb, *xempty = mb + 2, *yfull = mb + 4, *yempty = mb + 6;
  // S -> E: row e2's ring values are in place (rfull[e2 & 1]); E -> S: its runs are written
  // (rfree[e2 & 1]).  Two barriers each: the S warps may be two rows ahead of the emitters.
  uint64_t *rfull = mb + 8, *rfree = mb + 10;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(rfull + b, NWS * 32);
      mbar_init(rfree + b, NWE * 32);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(xfull + b, NWA * 32);
      mbar_init(xempty + b, NWB * 32);
      mbar_init(yfull + b, NWB * 32);
      mbar_init(yempty + b, NWS * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < Q) wq[tid] = a.weights[tid];
  if (N <= NBT) {
    int2* bt = reinterpret_cast<int2*>(sm + OFF_BT);
    for (int I = tid; I < N; I += NT) bt[I] = make_int2((int)band_prefix(I, P, N), (int)band_cnt(I, P, N));
  }
  if (tid < NPEN) {
    const int64_t I0 = i00 + tid / TB, I1 = i10 + tid % TB;
    pb[tid] = (I0 < N && I1 < N) ? rowptr3(I0, I1, 0, P, N) - a.base : 0;
    pc[tid] = (I0 < N && I1 < N) ? (int)(band_cnt(I0, P, N) * band_cnt(I1, P, N)) : 0;
  }
  __syncthreads();
  // Scalar coefficient on the uniform mesh: W = c w0 w1 w2 jac (the reference's factor order)
  // is the same for every element column and formed once; with a general knot vector it is
  // formed per column by the A warps.  FOLD (the launcher's choice for a coefficient field):
  // the axis weights go into the constant fragments -- w0 into stage A's, w1 into stage B's,
  // w2 jac into stage S's per column -- and W is the raw coefficient, copied a column ahead
  // by the A warps with cp.async (no per-column weight pass on their critical path: a
  // coefficient field used to run the C3 shape in 2.24 ms against 0.43 for a scalar).
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
    // coefficient field: W is double-buffered, column it + 1 is copied while it is used
    double* W2 = sm + Rg<FOLD>::OFF_W2;
    if (FOLD) copy_coef_column(W, a, 0, i00, i10, e0lo, e0hi, tid, NWA * 32);
    for (int it = 0; it < K; ++it) {
      const int b = it & 1;
      if (!FOLD && w_per_step) {
        if (it > 0) asm volatile("bar.sync 1, %0;\n" ::"n"(NWA * 32));  // W of it-1 consumed
        form_w(W, wq, a, it, i00, i10, e0lo, e0hi, tid, NWA * 32);
        asm volatile("bar.sync 1, %0;\n" ::"n"(NWA * 32));
      }
      if (FOLD) {
        // this column's coefficients have landed, for every A warp, and every A warp is done
        // with the other buffer (column it - 1): the next column's copy starts
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        asm volatile("bar.sync 1, %0;\n" ::"n"(NWA * 32));
        if (it + 1 < K) copy_coef_column(b ? W : W2, a, it + 1, i00, i10, e0lo, e0hi, tid, NWA * 32);
      }
      const double* Wc = (FOLD && b) ? W2 : W;
      if (it >= 2) mbar_wait(xempty + b, ((it >> 1) - 1) & 1);
      double* X = sm + OFF_X + b * SZ_X;
      int mt = mt0;
      for (; mt + mstep < MT_A; mt += 2 * mstep) stage_a_units<2>(L, Wc, ba, X, mt, mstep, ty);
      if (mt < MT_A) stage_a_units<1>(L, Wc, ba, X, mt, mstep, ty);
      mbar_arrive(xfull + b);
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
      const int b = e2 & 1, n = e2 >> 1;
      mbar_wait(xfull + b, n & 1);
      if (n >= 1) mbar_wait(yempty + b, (n - 1) & 1);
      const double* X = sm + OFF_X + b * SZ_X;
      double* Y = sm + OFF_Y + b * SZ_Y;
      for (int u = wb; u < NHB; u += NWB) stage_b_half(L, X, bv, bd, Y, u >> 1, u & 1);
      mbar_arrive(xempty + b);
      mbar_arrive(yfull + b);
    }
  } else if (warp >= NWA + NWB + NWS) {
    // ------------------------------------------------------------ role E
    // the mirrored runs of target rows e2 (hi) and e2 - 3 (lo) leave once the S warps have put
    // row e2's values into their rings
    const int et = tid - (NWA + NWB + NWS) * 32;
    __syncthreads();  // the S warps have written their mirror metadata
    EMeta em;
#pragma unroll
    for (int j = 0; j < ENJ; ++j) {
      const int c = (et >> 2) + j * ENG;
      em.row[j] = a.values; em.cx[j] = 0; em.cy[j] = -1;
      if (c < NRC) {
        const int2 cb = *reinterpret_cast<const int2*>(sm + OFF_MM + 2 * c + 1);
        em.row[j] = a.values + *reinterpret_cast<const int64_t*>(sm + OFF_MM + 2 * c);
        em.cx[j] = cb.x; em.cy[j] = cb.y;
      }
    }
    for (int e2 = 0; e2 < N; ++e2) {
      mbar_wait(rfull + (e2 & 1), (e2 >> 1) & 1);
      emit_all<true, FOLD>(a, sm, em, et, e2, N);
      if (e2 >= 3) emit_all<false, FOLD>(a, sm, em, et, e2 - 3, N);
      mbar_arrive(rfree + (e2 & 1));
    }
    // lo runs of the last three target rows (their later sources do not exist)
    for (int J2 = max(0, (int)N - 3); J2 < N; ++J2) emit_all<false, FOLD>(a, sm, em, et, J2, N);
  } else {
    // ------------------------------------------------------------ role S
    const int ws = warp - NWA - NWB;
    // per-lane store metadata of its m-tiles: pencil rc and the (d0,d1) block offset
    // b01 = (d0-lo0)*c1 + (d1-lo1) in the CSR row; -1 if the combo is outside
    int meta[MT_S_PER_WARP];
    double* mmw = sm + OFF_MM + 2 * (ws * MT_S_PER_WARP * 8 + L.g);  // its lane groups' mirror metadata
    double* rgw = sm + OFF_RING + ws * MT_S_PER_WARP * 8 * Rg<FOLD>::RING;  // this warp's rings
#pragma unroll
    for (int i = 0; i < MT_S_PER_WARP; ++i) {
      const int mt = ws + i * NWS;
      meta[i] = -1;
      if (mt < MT_S) {
        const int cb = mt * 8 + L.g;
        const int d1 = cb % NB, ib = (cb / NB) % TB, a0 = cb / (NB * TB);
        const int dh = a0 % NBH, ia = a0 / NBH, d0 = P + dh;
        const int I0 = i00 + ia, I1 = i10 + ib;
        int64_t mbase = 0;
        int mc01 = 0, mb01 = -1;
        if (I0 < a.plane_end && I1 < N) {
          const int lod0 = max(0, P - I0), lod1 = max(0, P - I1);
          const int c0 = (int)band_cnt(I0, P, N), c1 = (int)band_cnt(I1, P, N);
          if (d0 >= lod0 && d0 < lod0 + c0 && d1 >= lod1 && d1 < lod1 + c1) {
            meta[i] = ((ia * TB + ib) << 16) | ((d0 - lod0) * c1 + (d1 - lod1));
            if (dh > 0 && I0 + dh < a.plane_end) {
              // mirror: row J = (I0 + dh, I1 + d1 - P, .) holds this value at (P - dh, 2P - d1, .)
              // (a slab's J0 past its planes: the value is 0 there, no element of the slab
              // supports both rows)
              const int J0 = I0 + dh, J1 = I1 + d1 - P;
              const int jl0 = max(0, P - J0), jl1 = max(0, P - J1);
              const int jc1 = (int)band_cnt(J1, P, N);
              mbase = rowptr3(J0, J1, 0, P, N) - a.base;
              mc01 = (int)band_cnt(J0, P, N) * jc1;
              mb01 = (P - dh - jl0) * jc1 + (2 * P - d1 - jl1);
            }
          }
        }
        if (L.t == 0) {
          *reinterpret_cast<int64_t*>(mmw + i * 16) = mbase;
          *reinterpret_cast<int2*>(mmw + i * 16 + 1) = make_int2(mc01, mb01);
        }
      } else if (L.t == 0) {
        *reinterpret_cast<int2*>(mmw + i * 16 + 1) = make_int2(0, -1);
      }
    }
    double* Rs = sm + OFF_R;
    for (int u = ws * 32 + L.lane; u < MT_S * 4 * 2 * 32; u += NWS * 32) Rs[u] = 0.0;
    double sb0[2], sb1[2];
    s_fragments<FOLD>(L, a, 0, FOLD ? __dmul_rn(axis_w(wq, a.wt, 0, L.t, Q), a.jac) : 1.0, sb0, sb1);
    SRaw sraw;
    __syncthreads();
    for (int e2 = 0; e2 < K; ++e2) {
      const int b = e2 & 1;
      mbar_wait(yfull + b, (e2 >> 1) & 1);
      const double* Y = sm + OFF_Y + b * SZ_Y;
      if (e2 > 0) s_raw_form<FOLD>(L, sraw, sb0, sb1);
      switch (e2 & 3) {
        case 0: stage_s<0, FOLD>(L, ws, Y, Rs, a, e2, meta, pb, pc, N, sb0, sb1, rgw); break;
        case 1: stage_s<1, FOLD>(L, ws, Y, Rs, a, e2, meta, pb, pc, N, sb0, sb1, rgw); break;
        case 2: stage_s<2, FOLD>(L, ws, Y, Rs, a, e2, meta, pb, pc, N, sb0, sb1, rgw); break;
        default: stage_s<3, FOLD>(L, ws, Y, Rs, a, e2, meta, pb, pc, N, sb0, sb1, rgw); break;
      }
      if (e2 + 1 < K) s_raw_load<FOLD>(L, a, e2 + 1, FOLD ? __dmul_rn(axis_w(wq, a.wt, e2 + 1, L.t, Q), a.jac) : 1.0, sraw);
      mbar_arrive(yempty + b);
      mbar_arrive(rfull + b);  // role E writes the mirrored runs this row completes
    }
    // rows K .. K+P-1 received their last contribution from element K-1
    for (int I2 = K; I2 < N; ++I2) {
      constexpr int LAG = Rg<FOLD>::LAG;
      if (I2 >= LAG) mbar_wait(rfree + ((I2 - LAG) & 1), ((I2 - LAG) >> 1) & 1);
      flush_tail<FOLD>(L, ws, Rs, I2, meta, pb, pc, a, N, rgw);
      mbar_arrive(rfull + (I2 & 1));
    }
  }
}

}  // namespace p3s

int launch_gsf_p3s(const GsfArgs& a0, cudaStream_t s) {
  GsfArgs a = a0;
  const int64_t N = (int64_t)a.K + p3s::P;
  const int planes = a.plane_end - a.plane_begin;
  if (planes <= 0) return IGA_OK;
  const int tiles0 = (planes + p3s::TA - 1) / p3s::TA;
  a.tiles1 = (int)((N + p3s::TB - 1) / p3s::TB);
  const int64_t grid = (int64_t)tiles0 * a.tiles1;
  const bool fold = a.coef != nullptr;
  const size_t smem = fold ? p3s::Rg<true>::SMEM_BYTES : p3s::Rg<false>::SMEM_BYTES;
  cudaError_t e = smem_attr_once(reinterpret_cast<const void*>(fold ? p3s::k_gsf3_p3s<true> : p3s::k_gsf3_p3s<false>), smem);
  if (e != cudaSuccess) return check_cuda(e, "gsf_p3 smem attr");
  if (fold) p3s::k_gsf3_p3s<true><<<(unsigned)grid, p3s::NT, smem, s>>>(a);
  else p3s::k_gsf3_p3s<false><<<(unsigned)grid, p3s::NT, smem, s>>>(a);
  return check_cuda(cudaGetLastError(), "gsf_p3 launch");
}

}  // namespace iga

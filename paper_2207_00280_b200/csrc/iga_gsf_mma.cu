// Assembled sum factorization for every (p, q) on FP64 tensor cores (DMMA.8x8x4).
//
// Same mathematics, tiling and element-column streaming as the scalar generic
// kernel (iga_gsf.cu header): per element column e2 a CTA forms the weights W of
// its quadrature slab and runs the three contractions, each a small dense GEMM
// against the CTA's constant pair-product tables (invalid element/row pairs carry
// zeros, so the GEMMs need no data-dependent structure):
//
//   stage A: X_T[a0][col]        = sum_kk PA_T[a0][kk] W[kk][col]     (M = TA(2P+1),
//                                                                      N = cols, K = (TA+P) q)
//   stage B: Y[(a0,k2)][b1]      = sum_kk X[a0][kk][k2] PB[b1][kk]    (three products)
//   stage S: R[combo][(r,s)]    += sum_k2 Y[combo][k2] Z_e2[k2][(r,s)] (scattered into the
//                                                                      rolling rows)
//
// Warps take (m-tile, n-tile) items of each GEMM; operands are read from shared
// memory per k-step as DMMA fragments (lane (g,t): A[g][t], B[t][g]; out-of-range
// rows/columns/k predicated to zero, nothing is padded in memory), and the
// accumulators leave as the C fragments (C[g][2t], C[g][2t+1]).  k_gsf3_p3 keeps
// its hand-scheduled p = 3, q = 4 pipeline; this kernel serves the other degrees.
//
// Work the tiles do not need is not issued (C4, 96^3 p = 4 stiffness+mass with a
// coefficient field: 15.8 -> 11.8 ms; C2: 0.072 -> 0.059 ms):
//  * k-steps whose PA / PB fragment block is structurally zero (Band: an element of the
//    window supports both dofs of a row only in a band) are skipped, with compile-time
//    k-step ranges per tile and warps split across tiles by their nonzero work;
//  * stage S of the stiffness operators contracts [Y_A | Y_B] against [VV; DD] as one
//    K = 2q product (q = 5: 3 k-steps instead of 2 x 2), the rolling-row values being the
//    DMMA C operand, and the one or two (r, s) pairs past the last full n-tile (p = 2: 9
//    pairs, p = 4: 25) are summed with DFMAs instead of an n-tile that is 1/8 useful.
#include <cstdlib>
#include <type_traits>

#include "iga_args.cuh"
#include "iga_dispatch.cuh"

namespace iga {
bool sym_covers(const GsfArgs& a, int p);                // iga_gsf.cu
int sym_prezero(const GsfArgs& a, int p, cudaStream_t s);  // iga_gsf.cu
namespace mma {

// threads per CTA: 512 (one CTA per SM, shared-memory bound) for p >= 3; 256 for p <= 2, whose
// small tiles run four CTAs per SM (more element-column segments in flight for small meshes)
template <int P>
__host__ __device__ constexpr int nt_of() { return P <= 2 ? 256 : 512; }
__host__ __device__ constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }
// smallest pitch >= n with pitch == r (mod mod)
__host__ __device__ constexpr int pitch_mod(int n, int mod, int r) { return n + ((r - n % mod) % mod + mod) % mod; }
// Row order inside an 8-row DMMA m-tile so that the two rows (g = 2i, 2i+1) of each
// 16-byte quarter-warp phase sit `d` rows apart: for a row stride s (double2 units),
// d = 4 (s odd), 2 (s = 2, 6 mod 8), 1 (s = 4 mod 8) puts their 4 consecutive k-step
// columns in disjoint halves of the 8 bank groups (no shared-memory bank conflicts).
__host__ __device__ constexpr int qw_dist(int s) { return s % 2 ? 4 : (s % 4 == 2 ? 2 : 1); }
__device__ __forceinline__ int qw_row(int g, int d) {
  return d == 4 ? (g >> 1) + 4 * (g & 1) : (d == 2 ? (g & 4) + ((g >> 1) & 1) + 2 * (g & 1) : g);
}

// Structural zeros of the pair tables.  PA[a0][kk], a0 = (ia, d0), kk = (la, k0), is nonzero
// only if the element la of the window supports both dofs: r = ia + P - la and s = ia + d0 - la
// in [0, P] (PB the same with (ib, d1), (lb, k1)).  A DMMA k-step whose 8 x 4 fragment block is
// zero on every tile is skipped; the nonzero k-steps of each 8-row tile form one contiguous
// range [lo, hi) (C4, p = 4, TA = 1 / TB = 4: stage A 9 of 14 blocks, stage B 33 of 50).
// (NBX, D0X: the symmetric kernel keeps only the rows d = D0X .. D0X + NBX - 1 of each i)
template <int P, int Q, int T, int NBX = 2 * P + 1, int D0X = 0>
struct Band {
  static constexpr int NB = 2 * P + 1, KK = (T + P) * Q, ROWS = T * NBX;
  static constexpr int MT = cdiv(ROWS, 8), KS = cdiv(KK, 4);
  static constexpr bool nz(int mt, int ks) {
    for (int a = mt * 8; a < mt * 8 + 8 && a < ROWS; ++a)
      for (int kk = ks * 4; kk < ks * 4 + 4 && kk < KK; ++kk) {
        const int i = a / NBX, d = D0X + a % NBX, l = kk / Q, r = i + P - l, s = i + d - l;
        if (r >= 0 && r <= P && s >= 0 && s <= P) return true;
      }
    return false;
  }
  static constexpr int lo(int mt) {
#ifdef GSF_NOSKIP
    return 0;
#endif
    for (int ks = 0; ks < KS; ++ks)
      if (nz(mt, ks)) return ks;
    return KS;
  }
  static constexpr int hi(int mt) {
#ifdef GSF_NOSKIP
    return KS;
#endif
    for (int ks = KS; ks > 0; --ks)
      if (nz(mt, ks - 1)) return ks;
    return 0;
  }
};

// Warps per tile of a stage: every warp keeps one tile's constant fragments and sweeps
// `items` GEMM blocks of cost (hi - lo) k-steps; warps are added greedily to the tile with
// the largest per-warp load (tiles with fewer nonzero k-steps get fewer warps).
template <int MT>
struct Split {
  int cnt[MT];
  int start[MT + 1];
};
template <int MT, class B>
constexpr Split<MT> make_split(int nwarp, int items) {
  Split<MT> s{};
  for (int t = 0; t < MT; ++t) s.cnt[t] = 1;
  for (int used = MT; used < nwarp; ++used) {
    int best = -1, load = -1;
    for (int t = 0; t < MT; ++t) {
      const int l = cdiv(items, s.cnt[t]) * (B::hi(t) - B::lo(t));
      if (l > load) { load = l; best = t; }
    }
    if (s.cnt[best] >= items) break;
    ++s.cnt[best];
  }
  s.start[0] = 0;
  for (int t = 0; t < MT; ++t) s.start[t + 1] = s.start[t] + s.cnt[t];
  return s;
}
// this warp's tile, its index among the tile's warps, the tile's warp count and k-step range
// (tile -1: idle in this stage)
struct WarpTile {
  int tile = -1, grp = 0, cnt = 1, lo = 0, hi = 0;
};
template <int MT, class B, int NW, int ITEMS>
__device__ __forceinline__ WarpTile warp_tile(int warp) {
  static_assert(MT <= NW, "every tile needs at least one warp");
  constexpr Split<MT> s = make_split<MT, B>(NW, ITEMS);
  static_assert(s.start[MT] <= NW, "warp split exceeds the CTA");
  WarpTile w;
#pragma unroll
  for (int t = 0; t < MT; ++t)
    if (warp >= s.start[t] && warp < s.start[t + 1]) {
      w.tile = t; w.grp = warp - s.start[t]; w.cnt = s.cnt[t]; w.lo = B::lo(t); w.hi = B::hi(t);
    }
  return w;
}

// f(integral_constant<int, tile>) for the runtime tile index: the tile's k-step range is a
// compile-time constant inside f, so its fragment loads are unrolled and hoisted
template <int T, int MT, class F>
__device__ __forceinline__ void tile_dispatch(int tile, F&& f) {
  if constexpr (T < MT) {
    if (tile == T) f(std::integral_constant<int, T>());
    else tile_dispatch<T + 1, MT>(tile, f);
  }
}

// ST: stiffness (two operand types, double2 elements) or mass (one type: double elements,
// half the footprint of X, Y, PA, PB and Z, so p = 2 mass runs four CTAs per SM)
template <int P, int Q, int TA, int TB, bool ST = true, bool SYM = false>
struct Shape {
  static constexpr int EW = ST ? 2 : 1;
  static constexpr int m = P + 1, NB = 2 * P + 1;
  // axis-0 band offsets kept: all 2p+1, or (symmetric half) d0 = p .. 2p (J0 >= I0)
  static constexpr int NBX = SYM ? P + 1 : NB, D0X = SYM ? P : 0;
  static constexpr int LA = TA + P, LB = TB + P;
  static constexpr int KA = LA * Q, KB = LB * Q;  // contraction lengths of stages A, B
  static constexpr int GC = KB * Q;               // stage-A columns (k2, lb, k1), k2 slowest
  // conflict-free pitches: W rows (8-byte B fragments, 16-lane phases) == 4 mod 16
  // doubles; PA / PB rows (16-byte A / B fragments, 8-lane phases) == 4 mod 8 double2
  static constexpr int GCW = pitch_mod(GC, 16, 4);
  static constexpr int KAP = pitch_mod(KA, 8, 4), KBP = pitch_mod(KB, 8, 4);
  static constexpr int NA0 = TA * NBX, NB1 = TB * NB, NC = NA0 * NB1, NR = NA0 * Q;
  static constexpr int rowVals = NBX * NB * NB;  // values of a rolling row (the kept d0 blocks)
  // Y: mass [NC][Q] doubles; stiffness [NC][YPS] doubles, Y_A at k2 and Y_B at Q + k2, so
  // stage S runs its two products as one K = 2Q contraction (C4: 3 k-steps instead of 2 x 2);
  // YPS == 4 mod 8: the A fragments of a k-step (8 rows x 4 k) hit 16 distinct banks per phase
  static constexpr int YPS = ST ? pitch_mod(2 * Q, 8, 4) : Q;
  static constexpr int nW = KA * GCW, nY = NC * YPS;
  // Y aliases W (W is dead after stage A); even, so the double2 arrays after it are aligned
  static constexpr int nWY = ((nW > nY ? nW : nY) + 1) / 2 * 2;
  static constexpr int nX = EW * NA0 * GC;
  static constexpr int nPA = EW * NA0 * KAP, nPB = EW * NB1 * KBP;
  static constexpr int nZ = EW * m * m * Q;
  // rolling-row slot pitch: rowVals + a pad that spreads the stage-S read-modify-writes
  // over the shared-memory banks (picked by simulating the access pattern of the two
  // coefficient-field configs: 37% fewer wavefronts at p = 4, q = 5; 20% at p = 2, q = 3)
  static constexpr int RP = rowVals + (SYM                                      ? 0
                                       : P == 4 && Q == 5 && TA * TB == 4          ? 1
                                       : P == 2 && Q == 3 && TA == 3 && TB == 3 ? 7
                                                                                : 0);
  static constexpr int nR = TA * TB * m * RP;
  // symmetric half: the mirrored combos (d0 > p), per combo a ring of hi runs [m rows][m]
  // and lo runs [m rows][p] by target row; their mirror metadata; an axis-2 band table
  static constexpr int NRC = SYM ? TA * P * NB1 : 0, RING = m * NB;
  static constexpr int NBT = 1024;
  static constexpr int nRing = NRC * RING, nMM = 2 * NRC, nBT = SYM ? NBT : 0;
  static constexpr size_t bytes =
      sizeof(double) * ((size_t)nWY + nX + nPA + nPB + nZ + nR + nRing + nMM + nBT);
};

// shared-memory element of the operand tables: (V, D) pairs for stiffness, V only for mass
template <bool ST>
struct Elem {
  using T = double2;
  static __device__ __forceinline__ double2 mk(double x, double y) { return make_double2(x, y); }
};
template <>
struct Elem<false> {
  using T = double;
  static __device__ __forceinline__ double mk(double x, double) { return x; }
};
__device__ __forceinline__ double2 as2(double2 v) { return v; }
__device__ __forceinline__ double2 as2(double v) { return make_double2(v, 0.0); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

template <int P, int Q, int TA, int TB, bool STIFF, bool SYM>
__global__ void __launch_bounds__(nt_of<P>(), P <= 2 ? 4 : 1) k_gsf3_mma(GsfArgs a) {
  constexpr int NT = nt_of<P>();
  using S = Shape<P, Q, TA, TB, STIFF, SYM>;
  constexpr int NBX = S::NBX, D0X = S::D0X;
  using E = typename Elem<STIFF>::T;
  constexpr int m = S::m, NB = S::NB, KA = S::KA, KB = S::KB, GC = S::GC;
  constexpr int GCW = S::GCW, KAP = S::KAP, KBP = S::KBP;
  constexpr int NA0 = S::NA0, NB1 = S::NB1, NC = S::NC, NR = S::NR;
  extern __shared__ double smem[];
  double* sW = smem;                                         // [KA][GCW]
  double* Yd = smem;                                         // [NC][YPS] (aliases W)
  E* X2 = reinterpret_cast<E*>(smem + S::nWY);               // [NA0][Q][KB] (XV, XD)
  E* PA2 = X2 + NA0 * GC;                                    // [NA0][KAP] (VV, DD)
  E* PB2 = PA2 + NA0 * KAP;                                  // [NB1][KBP] (VV, DD)
  E* Z2 = PB2 + NB1 * KBP;                                   // [Q][m*m] (VV, DD(+VV))
  double* R = reinterpret_cast<double*>(Z2 + m * m * Q);     // [TA*TB][m][RP]
  double* RG = R + S::nR;                                    // [NRC][RING] mirror rings
  double* MM = RG + S::nRing;                                // [NRC] {int64 base, int2 {c01, b01}}
  int2* BT = reinterpret_cast<int2*>(MM + S::nMM);           // [NBT] {band_prefix, band_cnt}
  __shared__ int64_t rowoff[TA * TB];
  __shared__ int comboR[NC];  // R offset of combo (a0, b1): pencil block + (d0, d1) row

  const int K = a.K;
  const int64_t N = (int64_t)K + P;
  const int tile = blockIdx.x / a.segs, seg = blockIdx.x % a.segs;
  const int tile0 = tile / a.tiles1, tile1 = tile % a.tiles1;
  const int i00 = a.plane_begin + tile0 * TA, i10 = tile1 * TB;
  const int s0 = seg * a.seg_len, s1 = min(K, s0 + a.seg_len);
  const int e_first = max(0, s0 - P);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, g = lane >> 2, t = lane & 3;
  constexpr int NWARP = NT / 32;
  const int e0lo = max(a.el_begin, 0), e0hi = min(a.el_end, K);
  const double* V = a.V;
  const double* D = a.D;

  // ---- constant pair tables (axis 0 slab-restricted, axis 1)
  for (int u = tid; u < NA0 * KA; u += NT) {
    const int a0 = u / KA, kk = u % KA, la = kk / Q, k0 = kk % Q;
    const int I0 = i00 + a0 / NBX, J0 = I0 - P + D0X + a0 % NBX, e0 = i00 - P + la;
    const int r = I0 - e0, sc = J0 - e0;
    double2 v = make_double2(0.0, 0.0);
    if (e0 >= e0lo && e0 < e0hi && r >= 0 && r <= P && sc >= 0 && sc <= P && J0 >= 0 && J0 < N) {
      v.x = V[((int64_t)e0 * m + r) * Q + k0] * V[((int64_t)e0 * m + sc) * Q + k0];
      if (STIFF) v.y = D[((int64_t)e0 * m + r) * Q + k0] * D[((int64_t)e0 * m + sc) * Q + k0];
#ifndef GSF_NOFOLD
      // the axis-0 weight lives in the pair table (W is the raw coefficient, below)
      const double w0 = axis_w(a.weights, a.wt, e0, k0, Q);
      v.x = __dmul_rn(v.x, w0);
      v.y = __dmul_rn(v.y, w0);
#endif
    }
    PA2[a0 * KAP + kk] = Elem<STIFF>::mk(v.x, v.y);
  }
  for (int u = tid; u < NB1 * KB; u += NT) {
    const int b1 = u / KB, kk = u % KB, lb = kk / Q, k1 = kk % Q;
    const int I1 = i10 + b1 / NB, J1 = I1 - P + b1 % NB, e1 = i10 - P + lb;
    const int r = I1 - e1, sc = J1 - e1;
    double2 v = make_double2(0.0, 0.0);
    if (e1 >= 0 && e1 < K && r >= 0 && r <= P && sc >= 0 && sc <= P && J1 >= 0 && J1 < N) {
      v.x = V[((int64_t)e1 * m + r) * Q + k1] * V[((int64_t)e1 * m + sc) * Q + k1];
      if (STIFF) v.y = D[((int64_t)e1 * m + r) * Q + k1] * D[((int64_t)e1 * m + sc) * Q + k1];
#ifndef GSF_NOFOLD
      const double w1 = axis_w(a.weights, a.wt, e1, k1, Q);
      v.x = __dmul_rn(v.x, w1);
      v.y = __dmul_rn(v.y, w1);
#endif
    }
    PB2[b1 * KBP + kk] = Elem<STIFF>::mk(v.x, v.y);
  }
  for (int u = tid; u < S::nR; u += NT) R[u] = 0.0;
  for (int c = tid; c < NC; c += NT) {
    const int a0 = c / NB1, b1 = c % NB1;
    const int ia = a0 / NBX, dx = a0 % NBX, ib = b1 / NB, d1 = b1 % NB;
    comboR[c] = (ia * TB + ib) * m * S::RP + (dx * NB + d1) * NB;
  }
  if constexpr (SYM) {
    // mirror metadata of combo c = ((ia p + dx - 1) TB + ib) NB + d1 (d0 = p + dx > p): the
    // value at (I, J) also belongs at (J, I), J = (I0 + dx, I1 + d1 - p, .), whose row holds
    // it at block (p - dx, 2p - d1); b01 -1: no mirror
    for (int c = tid; c < S::NRC; c += NT) {
      const int d1 = c % NB, ib = (c / NB) % TB, dx = 1 + (c / (NB * TB)) % P, ia = c / (NB * TB * P);
      const int I0 = i00 + ia, I1 = i10 + ib, J0 = I0 + dx, J1 = I1 - P + d1;
      int64_t base = 0;
      int c01 = 0, b01 = -1;
      // (a slab's J0 past its planes: the value is 0 there, no element of the slab supports both rows)
      if (I0 < a.plane_end && I1 < N && J0 < a.plane_end && J0 < N && J1 >= 0 && J1 < N) {
        const int jc1 = (int)band_cnt(J1, P, N);
        base = rowptr3(J0, J1, 0, P, N) - a.base;
        c01 = (int)band_cnt(J0, P, N) * jc1;
        b01 = (P - dx - max(0, P - J0)) * jc1 + (2 * P - d1 - max(0, P - J1));
      }
      *reinterpret_cast<int64_t*>(MM + 2 * c) = base;
      *reinterpret_cast<int2*>(MM + 2 * c + 1) = make_int2(c01, b01);
    }
    if (N <= S::NBT)
      for (int I = tid; I < N; I += NT) BT[I] = make_int2((int)band_prefix(I, P, N), (int)band_cnt(I, P, N));
  }

  // W units: one (kk, (lb, k1)) row segment of Q contiguous k2 columns per unit (the Q
  // coefficients of a unit are contiguous in memory); the thread's units are fixed, and
  // their coefficients for the next element column are prefetched into registers
  constexpr int NUW = KA * KB, UPT = cdiv(NUW, NT), Q3 = Q * Q * Q;
  // per-axis weights of the tile's element windows (axis 0: la, axis 1: lb) and of the
  // current column e2: the reference weights, or for a general knot vector the per-element
  // tables w_k h_e / 2 (out-of-mesh window elements: 0, their pair tables are 0 as well)
  __shared__ double wqs[Q], wa[KA], wb[KB];
  if (tid < Q) wqs[tid] = a.weights[tid];
  for (int u = tid; u < KA + KB; u += NT) {
    const bool ax0 = u < KA;
    const int v = ax0 ? u : u - KA, l = v / Q, k = v % Q;
    const int e = ax0 ? i00 - P + l : i10 - P + l;
    const double w = a.wt == nullptr ? a.weights[k] : (e >= 0 && e < K ? __ldg(a.wt + e * Q + k) : 0.0);
    if (ax0) wa[v] = w; else wb[v] = w;
  }
  // per unit: the coefficient offset without the e2 term (-1: out of the mesh) and the W row
  // offset, computed once
  int64_t cbase[UPT];
  int wdst[UPT];
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const int u = tid + i * NT;
    cbase[i] = -1;
    wdst[i] = -1;
    if (u < NUW) {
      const int kk = u / KB, c1 = u - kk * KB, la = kk / Q, k0 = kk - la * Q;
      const int lb = c1 / Q, k1 = c1 - lb * Q;
      const int e0 = i00 - P + la, e1 = i10 - P + lb;
      wdst[i] = kk * GCW + c1;
      if (e0 >= 0 && e0 < K && e1 >= 0 && e1 < K)
        cbase[i] = ((int64_t)e0 * K + e1) * K * Q3 + (k0 * Q + k1) * Q;
    }
  }
  auto load_coef = [&](int e2, double (&cv)[UPT][Q]) {
#pragma unroll
    for (int i = 0; i < UPT; ++i) {
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) cv[i][k2] = a.coef_scalar;
      if (a.coef && cbase[i] >= 0 && e2 < K) {
        const double* src = a.coef + cbase[i] + (int64_t)e2 * Q3;
#pragma unroll
        for (int k2 = 0; k2 < Q; ++k2) cv[i][k2] = __ldg(src + k2);
      }
    }
  };
  double cv[UPT][Q];
  load_coef(e_first, cv);
  // axis-2 table entries of the next element (one (r, s, k) per thread)
  static_assert(m * m * Q <= NT, "one Z entry per thread");
  auto load_z = [&](int e2, double (&zv)[4]) {
    zv[0] = zv[1] = zv[2] = zv[3] = 0.0;
    if (tid < m * m * Q && e2 < K) {
      const int k = tid / (m * m), n = tid % (m * m), r = n / m, sc = n % m;
      const double* V2 = V + (int64_t)e2 * m * Q;
      zv[0] = __ldg(V2 + r * Q + k);
      zv[1] = __ldg(V2 + sc * Q + k);
      if (STIFF) {
        const double* D2 = D + (int64_t)e2 * m * Q;
        zv[2] = __ldg(D2 + r * Q + k);
        zv[3] = __ldg(D2 + sc * Q + k);
      }
    }
  };
  double zv[4];
  load_z(e_first, zv);

  // a finished row leaves (and its slot is cleared) in the next column's stage-A phase, so
  // the row store costs no barrier of its own
  // per pencil rc of the row being flushed: CSR offset (-1: not written here) and, for
  // rows with a truncated band, the packed (lod0, lod1, c0, c1); 0 marks a full band
  __shared__ int rowmeta[TA * TB];
  auto set_rowoff = [&](int I2) {
    if (tid < TA * TB) {
      const int ia = tid / TB, ib = tid % TB;
      const int I0 = i00 + ia, I1 = i10 + ib;
      const bool ok = I2 >= s0 && I0 < a.plane_end && I1 < N;
      rowoff[tid] = ok ? rowptr3(I0, I1, I2, P, N) - a.base : -1;
      const bool full = I0 >= P && I0 < K && I1 >= P && I1 < K && I2 >= P && I2 < K;
      rowmeta[tid] = full ? 0
                          : 1 | max(0, P - I0) << 1 | max(0, P - I1) << 6 |
                                (int)band_cnt(I0, P, N) << 11 | (int)band_cnt(I1, P, N) << 16;
    }
  };
  // Row flush by (band position v, pencil rc).  When a row's band padded to whole warps
  // divides the CTA (p <= 2: 125 -> 128 lanes, two pencils per pass), every thread keeps one
  // v and its (d0, d1, d2) for the whole flush and walks the pencils; otherwise the flat
  // (rc, v) loop below.  Both write the same values to the same addresses.
  constexpr int VT = cdiv(S::rowVals, 32) * 32, RCS = NT / VT;
  constexpr bool by_v = !SYM && RCS >= 1 && RCS * VT == NT;
  // The flat flush shares its barrier phase with stage A.  Where stage A is one m-tile whose
  // n-tiles give the first NHV warps two and the others one (symmetric p = 4: 25 n-tiles, 16
  // warps), the other warps flush (GSF_REV & 4); else the band positions are dealt from the
  // last warp down (GSF_REV & 1), so the warps left without flush work are the first ones.
#ifndef GSF_REV
#define GSF_REV 7
#endif
  constexpr int NTL_A = cdiv(GC, 8), NWARP_ = NT / 32;
  constexpr bool split_flush = (GSF_REV & 4) && SYM && cdiv(NA0, 8) == 1 && NTL_A > NWARP_ && NTL_A < 2 * NWARP_;
  constexpr int NHV = split_flush ? NTL_A - NWARP_ : 0;  // warps with two stage-A n-tiles
  constexpr int NFT = NT - 32 * NHV;                      // flushing threads
  constexpr int VPT = cdiv(S::rowVals, NFT);
  const int FT = split_flush ? (tid >= 32 * NHV ? tid - 32 * NHV : S::rowVals) : (GSF_REV & 1) ? NT - 1 - tid : tid;
  int vd[VPT];  // (d0 - D0X, d1, d2) of this thread's band positions, packed
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int v = FT + j * NFT;
    vd[j] = (v / (NB * NB)) << 16 | ((v / NB) % NB) << 8 | (v % NB);
  }
  auto flush_row = [&](int I2) {
    const int slot = I2 % m;
    const int lod2 = max(0, P - I2), c2 = (int)band_cnt(I2, P, N);
    if constexpr (by_v) {
      const int v = tid % VT;
      if (v >= S::rowVals) return;
      double* Rv = R + slot * S::RP + v;
      if (I2 < s0) {  // recomputed halo row of this segment: nothing is written here
        for (int rc = tid / VT; rc < TA * TB; rc += RCS) Rv[rc * m * S::RP] = 0.0;
        return;
      }
      const int d2 = v % NB, d1 = (v / NB) % NB, d0 = v / (NB * NB);
      const bool in2 = d2 >= lod2 && d2 < lod2 + c2;
      for (int rc = tid / VT; rc < TA * TB; rc += RCS) {
        double* Rr = Rv + rc * m * S::RP;
        const int64_t off = rowoff[rc];
        if (off >= 0) {
          const int mt = rowmeta[rc];
          if (mt == 0) {
            a.values[off + v] = *Rr;
          } else {
            const int lod0 = (mt >> 1) & 31, lod1 = (mt >> 6) & 31, c0 = (mt >> 11) & 31,
                      c1 = (mt >> 16) & 31;
            if (in2 && d0 >= lod0 && d0 < lod0 + c0 && d1 >= lod1 && d1 < lod1 + c1)
              a.values[off + ((d0 - lod0) * c1 + (d1 - lod1)) * c2 + (d2 - lod2)] = *Rr;
          }
        }
        *Rr = 0.0;
      }
      return;
    }
    // otherwise every thread keeps its band positions v = tid + j NT (decomposed once) and
    // walks the pencils
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const int v = FT + j * NFT;
      if (v >= S::rowVals) break;
      const int d2 = vd[j] & 255, d1 = (vd[j] >> 8) & 255, dx = vd[j] >> 16, d0 = D0X + dx;
      const bool in2 = d2 >= lod2 && d2 < lod2 + c2;
      // symmetric half: target row J2 of this value's mirror and its ring entry
      const int J2 = I2 + d2 - P, d2p = 2 * P - d2;
      const int rg_off = J2 % m * (d2p <= P ? m : P) + (d2p <= P ? d2p : m * m + d2p - m);
#pragma unroll
      for (int rc = 0; rc < TA * TB; ++rc) {
        double* Rv = R + (rc * m + slot) * S::RP + v;
        const double val = *Rv;
        const int64_t off = rowoff[rc];
        if (off >= 0) {
          const int mt = rowmeta[rc];
          if (mt == 0) {
            a.values[off + D0X * NB * NB + v] = val;  // full band: CSR order is the R order
          } else {
            const int lod0 = (mt >> 1) & 31, lod1 = (mt >> 6) & 31, c0 = (mt >> 11) & 31,
                      c1 = (mt >> 16) & 31;
            if (in2 && d0 >= lod0 && d0 < lod0 + c0 && d1 >= lod1 && d1 < lod1 + c1)
              a.values[off + ((d0 - lod0) * c1 + (d1 - lod1)) * c2 + (d2 - lod2)] = val;
          }
        }
        if constexpr (SYM) {
          if (dx > 0 && J2 >= 0 && J2 < N) {
            const int c = (((rc / TB) * P + dx - 1) * TB + rc % TB) * NB + d1;
            RG[c * S::RING + rg_off] = val;
          }
        }
        *Rv = 0.0;
      }
    }
  };
  // Symmetric half: target row J2's complete mirror runs, hi (d2' = 0..p, complete once its
  // source row J2 is flushed) or lo (d2' = p+1..2p, once J2 + p is), one thread per (combo,
  // entry): consecutive threads write consecutive values of a run.  Only entries whose source
  // row this CTA writes (its segment) leave here.
  auto emit = [&](int J2, bool hi) {
    if constexpr (SYM) {
      if (J2 < 0 || J2 >= N) return;
      const int2 bq = N <= S::NBT ? BT[J2] : make_int2((int)band_prefix(J2, P, N), (int)band_cnt(J2, P, N));
      const int lod2 = max(0, P - J2), slot = J2 % m, ne = hi ? m : P;
      const int s1w = s1 == K ? (int)N : s1;
      for (int u = tid; u < S::NRC * ne; u += NT) {
        const int c = u / ne, e = u - c * ne, d2p = hi ? e : m + e;
        const int I2s = J2 - P + d2p;  // source row of the entry
        const int off = d2p - lod2;
        if (I2s < s0 || I2s >= s1w || off < 0 || off >= bq.y) continue;
        const int2 cb = *reinterpret_cast<const int2*>(MM + 2 * c + 1);
        if (cb.y < 0) continue;
        const int64_t base = *reinterpret_cast<const int64_t*>(MM + 2 * c);
        a.values[base + (int64_t)cb.x * bq.x + (int64_t)cb.y * bq.y + off] =
            RG[c * S::RING + (hi ? slot * m + e : m * m + slot * P + e)];
      }
    }
  };
  int pending = -1;
  for (int e2 = e_first; e2 < s1; ++e2) {
    __syncthreads();  // previous column's stage S (reads Y, aliasing W) is done
    if (pending >= 0) set_rowoff(pending);
#ifdef GSF_ABL_W
    if (e2 < 0)
#endif
    {
#ifndef GSF_NOFOLD
      // W is the raw coefficient: the axis weights live in the pair tables (w0 in PA, w1 in
      // PB) and in this column's Z (w2 jac), so the weight pass is a copy of the prefetched
      // coefficients (it was 22% of the C4 kernel with three multiplies and three weight
      // lookups per value)
#pragma unroll
      for (int i = 0; i < UPT; ++i) {
        if (wdst[i] >= 0) {
          double* dst = sW + wdst[i];  // column (k2, c1): k2 slowest
#pragma unroll
          for (int k2 = 0; k2 < Q; ++k2) dst[k2 * KB] = cv[i][k2];
        }
      }
#else
      double w2[Q];  // axis-2 weights of this column
#pragma unroll
      for (int k2 = 0; k2 < Q; ++k2) w2[k2] = axis_w(wqs, a.wt, e2, k2, Q);
#pragma unroll
      for (int i = 0; i < UPT; ++i) {  // W = ((w0 w1) w2) jac c, the reference's factor order
        if (wdst[i] >= 0) {
          const int u = tid + i * NT, kk = u / KB, c1 = u - kk * KB;
          const double w01 = wa[kk] * wb[c1];
          double* dst = sW + wdst[i];  // column (k2, c1): k2 slowest
#pragma unroll
          for (int k2 = 0; k2 < Q; ++k2) dst[k2 * KB] = w01 * w2[k2] * a.jac * cv[i][k2];
        }
      }
#endif
    }
    load_coef(e2 + 1, cv);
    if (tid < m * m * Q) {  // Z[k2][(r,s)]
#ifndef GSF_NOFOLD
      const double ws = __dmul_rn(axis_w(wqs, a.wt, e2, tid / (m * m), Q), a.jac);
      const double vv = __dmul_rn(zv[0], zv[1]);
      double dd = 0.0;
      if (STIFF) {
        dd = __dmul_rn(zv[2], zv[3]);
        if (a.op == IGA_OP_STIFFNESS_MASS) dd = __dadd_rn(dd, vv);
      }
      Z2[tid] = Elem<STIFF>::mk(__dmul_rn(vv, ws), __dmul_rn(dd, ws));
#else
      const double vv = zv[0] * zv[1];
      double dd = 0.0;
      if (STIFF) {
        dd = zv[2] * zv[3];
        if (a.op == IGA_OP_STIFFNESS_MASS) dd += vv;
      }
      Z2[tid] = Elem<STIFF>::mk(vv, dd);
#endif
    }
    load_z(e2 + 1, zv);
    __syncthreads();

#ifndef GSF_ABL_F  // ablation knob (tools/gsf_variants.sh): skip the row flush
    if (pending >= 0) flush_row(pending);
#endif
    // ---- stage A: X_T[a0][col] = sum_kk PA_T[a0][kk] W[kk][col]; warp w keeps the PA
    // fragments of m-tile w % MT in registers and sweeps its n-tiles
#ifdef GSF_ABL_A
    if (e2 < 0)
#endif
    {
      using BA = Band<P, Q, TA, NBX, D0X>;
      constexpr int MT = cdiv(NA0, 8), NTL = cdiv(GC, 8), KS = cdiv(KA, 4);
      static_assert(BA::MT == MT && BA::KS == KS, "stage-A band shape");
      const WarpTile wt = warp_tile<MT, BA, NWARP, NTL>(warp);
      tile_dispatch<0, MT>(wt.tile, [&](auto tc) {
        constexpr int LO = BA::lo(decltype(tc)::value), HI = BA::hi(decltype(tc)::value);
        const int row = decltype(tc)::value * 8 + g;
        double2 pa[HI - LO];
#pragma unroll
        for (int ks = LO; ks < HI; ++ks) {
          const int kk = ks * 4 + t;
          pa[ks - LO] = (row < NA0 && kk < KA) ? as2(PA2[row * KAP + kk]) : make_double2(0.0, 0.0);
        }
        for (int ntl = wt.grp; ntl < NTL; ntl += wt.cnt) {
          const int col = ntl * 8 + g;
          double cv0 = 0.0, cv1 = 0.0, cd0 = 0.0, cd1 = 0.0;
#pragma unroll
          for (int ks = LO; ks < HI; ++ks) {  // structurally zero k-steps skipped
            const int kk = ks * 4 + t;
            const double w = (kk < KA && col < GC) ? sW[kk * GCW + col] : 0.0;
            dmma(cv0, cv1, pa[ks - LO].x, w);
            if (STIFF) dmma(cd0, cd1, pa[ks - LO].y, w);
          }
          const int c0 = ntl * 8 + 2 * t;
          if (row < NA0) {
            if (c0 < GC) X2[row * GC + c0] = Elem<STIFF>::mk(cv0, cd0);
            if (c0 + 1 < GC) X2[row * GC + c0 + 1] = Elem<STIFF>::mk(cv1, cd1);
          }
        }
      });
    }
    __syncthreads();

    if constexpr (SYM) {
      if (pending >= 0) {  // the row flushed in this column's stage-A phase
        emit(pending, true);
        emit(pending - P, false);
      }
    }
    // ---- stage B: rows (a0, k2), columns b1; warp w keeps the PB fragments of n-tile
    // w % NTL in registers:  mass YA = XV VV;  stiffness YA = XV DD + XD VV, YB = XV VV
#ifdef GSF_ABL_B
    if (e2 < 0)
#endif
    {
      using BB = Band<P, Q, TB>;
      constexpr int MT = cdiv(NR, 8), NTL = cdiv(NB1, 8), KS = cdiv(KB, 4);
      static_assert(BB::MT == NTL && BB::KS == KS, "stage-B band shape");
      const WarpTile wt = warp_tile<NTL, BB, NWARP, MT>(warp);
      tile_dispatch<0, NTL>(wt.tile, [&](auto tc) {
        constexpr int LO = BB::lo(decltype(tc)::value), HI = BB::hi(decltype(tc)::value);
        const int ntl = decltype(tc)::value, b1 = ntl * 8 + g;
        constexpr int DQ = qw_dist(KB);  // X rows (a0, k2) are KB double2 apart
        double2 pb[HI - LO];
#pragma unroll
        for (int ks = LO; ks < HI; ++ks) {
          const int kk = ks * 4 + t;
          pb[ks - LO] = (b1 < NB1 && kk < KB) ? as2(PB2[b1 * KBP + kk]) : make_double2(0.0, 0.0);
        }
        for (int mt = wt.grp; mt < MT; mt += wt.cnt) {
          const int row = mt * 8 + qw_row(g, DQ), a0 = row / Q, k2 = row % Q;
          double ya0 = 0.0, ya1 = 0.0, yb0 = 0.0, yb1 = 0.0;
#pragma unroll
          for (int ks = LO; ks < HI; ++ks) {  // structurally zero k-steps skipped
            const int kk = ks * 4 + t;
            const double2 x = (row < NR && kk < KB) ? as2(X2[row * KB + kk]) : make_double2(0.0, 0.0);
            if (STIFF) {
              dmma(ya0, ya1, x.x, pb[ks - LO].y);
              dmma(ya0, ya1, x.y, pb[ks - LO].x);
              dmma(yb0, yb1, x.x, pb[ks - LO].x);
            } else {
              dmma(ya0, ya1, x.x, pb[ks - LO].x);
            }
          }
          const int c0 = ntl * 8 + 2 * t;
          if (row < NR) {
            constexpr int YPS = S::YPS;
            if (c0 < NB1) {
              Yd[(a0 * NB1 + c0) * YPS + k2] = ya0;
              if (STIFF) Yd[(a0 * NB1 + c0) * YPS + Q + k2] = yb0;
            }
            if (c0 + 1 < NB1) {
              Yd[(a0 * NB1 + c0 + 1) * YPS + k2] = ya1;
              if (STIFF) Yd[(a0 * NB1 + c0 + 1) * YPS + Q + k2] = yb1;
            }
          }
        }
      });
    }
    __syncthreads();

    // ---- stage S: C[combo][(r,s)] = sum_k2 Y[combo][k2] Z[k2][(r,s)] into the rolling
    // rows; warp w keeps the Z fragments of n-tile w % NTL and its lanes' two (r,s)
    // destinations, and sweeps the combo m-tiles
#ifdef GSF_ABL_S
    if (e2 < 0)
#endif
    {
      // n-tiles of (r, s) pairs; one or two pairs left over past the last full n-tile
      // (p = 2: 9 pairs, p = 4: 25) are summed with DFMAs below instead of a DMMA tile that
      // is 1/8 or 2/8 useful
      constexpr int MM = m * m, MT = cdiv(NC, 8), KQ = STIFF ? 2 * Q : Q, KS = cdiv(KQ, 4);
      constexpr int YPS = S::YPS;
#ifndef GSF_NOLEFT
      constexpr int NTL = (MM > 8 && MM % 8 != 0 && MM % 8 <= 2) ? MM / 8 : cdiv(MM, 8);
#else
      constexpr int NTL = cdiv(MM, 8);
#endif
      constexpr int GRP = NWARP / NTL;
      const int slot0 = e2 % m;
      if (warp < NTL * GRP) {
        const int ntl = warp % NTL, grp = warp / NTL, n = ntl * 8 + g;
        // B fragments: k < Q value products (VV), Q <= k < 2Q derivative products (DD (+VV))
#ifndef GSF_NOSTACK
        double z[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const int k = ks * 4 + t;
          const double2 zz = (n < MM && k < KQ) ? as2(Z2[(k < Q ? k : k - Q) * MM + n]) : make_double2(0.0, 0.0);
          z[ks] = k < Q ? zz.x : zz.y;
        }
#else
        constexpr int KS1 = cdiv(Q, 4);
        double2 z2[KS1];
#pragma unroll
        for (int ks = 0; ks < KS1; ++ks) {
          const int k = ks * 4 + t;
          z2[ks] = (n < MM && k < Q) ? as2(Z2[k * MM + n]) : make_double2(0.0, 0.0);
        }
#endif
        int dst[2];  // offset of column (r, s) in a combo's R block, -1 if padding
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int nn = ntl * 8 + 2 * t + j, r = nn / m, sc = nn % m;
          const int slot = slot0 + r >= m ? slot0 + r - m : slot0 + r;
          dst[j] = nn < MM ? slot * S::RP + sc - r + P : -1;
        }
        for (int mt = grp; mt < MT; mt += GRP) {
          const int combo = mt * 8 + g;
          const int cc = combo;  // C row = A row of this lane
          double* Rc = R + comboR[cc < NC ? cc : 0];
          // the rolling-row values are the C operand: R += Y Z in the DMMA itself
          double c0v = (cc < NC && dst[0] >= 0) ? Rc[dst[0]] : 0.0;
          double c1v = (cc < NC && dst[1] >= 0) ? Rc[dst[1]] : 0.0;
#ifndef GSF_NOSTACK
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const int k = ks * 4 + t;
            const double y = (combo < NC && k < KQ) ? Yd[combo * YPS + k] : 0.0;
            dmma(c0v, c1v, y, z[ks]);
          }
#else
#pragma unroll
          for (int ks = 0; ks < KS1; ++ks) {
            const int k = ks * 4 + t;
            const double ya = (combo < NC && k < Q) ? Yd[combo * YPS + k] : 0.0;
            dmma(c0v, c1v, ya, z2[ks].x);
            if (STIFF) {
              const double yb = (combo < NC && k < Q) ? Yd[combo * YPS + Q + k] : 0.0;
              dmma(c0v, c1v, yb, z2[ks].y);
            }
          }
#endif
          if (cc < NC) {
            if (dst[0] >= 0) Rc[dst[0]] = c0v;
            if (dst[1] >= 0) Rc[dst[1]] = c1v;
          }
        }
      }
      if constexpr (NTL * 8 < MM) {
        // leftover pairs: one (combo, pair) per thread, distinct R entries from the DMMA part
        constexpr int NL = MM - NTL * 8;
        // (dealt from the last warp down, GSF_REV & 2: the warps past NTL * GRP and those of
        // the last groups have the fewest m-tiles)
        for (int u = (GSF_REV & 2) ? NT - 1 - tid : tid; u < NC * NL; u += NT) {
          const int c = u / NL, nn = NTL * 8 + u % NL, r = nn / m, sc = nn % m;
          const int slot = slot0 + r >= m ? slot0 + r - m : slot0 + r;
          double* Rr = R + comboR[c] + slot * S::RP + sc - r + P;
          double acc = *Rr;
#pragma unroll
          for (int k = 0; k < KQ; ++k) {
            const double2 zz = as2(Z2[(k < Q ? k : k - Q) * MM + nn]);
            acc = fma(Yd[c * YPS + k], k < Q ? zz.x : zz.y, acc);
          }
          *Rr = acc;
        }
      }
    }

    pending = e2;  // row e2 has its last contribution; written during the next column
  }
  // rows still in flight: the last column's row and, after element K-1, rows K .. N-1
  if (pending >= 0) {
    const int last = (pending == K - 1) ? (int)N - 1 : pending;
    for (int I2 = pending; I2 <= last; ++I2) {
      __syncthreads();
      set_rowoff(I2);
      __syncthreads();
      flush_row(I2);
      if constexpr (SYM) {
        __syncthreads();
        emit(I2, true);
        emit(I2 - P, false);
      }
    }
    if constexpr (SYM) {
      // runs this CTA's last rows feed but never completed here: the lo runs of the last p
      // target rows and, before the next segment, the hi runs of the p rows after it (the
      // entries of other segments' source rows are theirs)
      for (int J2 = last + 1 - P; J2 <= last; ++J2) emit(J2, false);
      for (int J2 = last + 1; J2 <= last + P; ++J2) emit(J2, true);
    }
  }
}

// Tile of row pencils per CTA: 3 x 3 for p = 2 (stage-A rows 15 of 16 and stage-B columns
// 15 of 16 in their DMMA tiles; C2 32^3: 144 tiles, 0.087 vs 0.099 ms with 2 x 4), 1 x 4 for
// p = 4 (7% fewer DMMAs per pencil than 2 x 2; C4 16.0 vs 16.3 ms), else the largest of
// 2 x 4 / 2 x 2 / 2 x 1 / 1 x 1 that fits shared memory
template <int P, int Q, bool ST>
struct Tile {
  static constexpr size_t cap = 227 * 1024;
  static constexpr bool t33 = P == 2 && Shape<P, Q, 3, 3, ST>::bytes <= cap;
  static constexpr bool t14 = P == 4 && Shape<P, Q, 1, 4, ST>::bytes <= cap;
  static constexpr int TA = t33 ? 3
                            : t14 ? 1
                            : Shape<P, Q, 2, 4, ST>::bytes <= cap ? 2
                            : Shape<P, Q, 2, 2, ST>::bytes <= cap ? 2
                            : Shape<P, Q, 2, 1, ST>::bytes <= cap ? 2 : 1;
  static constexpr int TB = t33 ? 3
                            : t14 ? 4
                            : Shape<P, Q, 2, 4, ST>::bytes <= cap ? 4
                            : Shape<P, Q, 2, 2, ST>::bytes <= cap ? 2 : 1;
};

template <int P, int Q, bool ST, bool SYM = false, int TA = Tile<P, Q, ST>::TA, int TB = Tile<P, Q, ST>::TB>
static int launch_t(const GsfArgs& a0, cudaStream_t s) {
  using Sh = Shape<P, Q, TA, TB, ST, SYM>;
  if constexpr (SYM && Sh::bytes > 227 * 1024) {
    return launch_t<P, Q, ST, false>(a0, s);  // the symmetric half's rings do not fit
  } else if constexpr (Sh::bytes > 227 * 1024) {
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
    const void* fn = reinterpret_cast<const void*>(k_gsf3_mma<P, Q, TA, TB, ST, SYM>);
    cudaError_t e = smem_attr_once(fn, Sh::bytes, true);
    if (e != cudaSuccess) return check_cuda(e, "gsf mma smem attr");
    constexpr int NT = nt_of<P>();
    const int64_t slots = (int64_t)sm_count() * blocks_per_sm_once(fn, NT, Sh::bytes);
    int best = 1;
    double best_cost = 1e300;
    static const int force_segs = [] {  // tuning knob: force the segment count (read once)
      const char* es = getenv("IGA_GSF_SEGS");
      return es && *es ? atoi(es) : 0;
    }();
    for (int sg = 1; sg <= a.K; ++sg) {
      if (force_segs > 0 && sg != force_segs) continue;
      const int L = (a.K + sg - 1) / sg;
      if (L < P && sg > 1) break;
      const double waves = (double)((tiles * sg + slots - 1) / slots);
      const double cost = waves * (L + (sg > 1 ? P : 0));
      if (cost < best_cost - 1e-9) { best_cost = cost; best = sg; }
    }
    a.segs = best;
    a.seg_len = (a.K + best - 1) / best;
    k_gsf3_mma<P, Q, TA, TB, ST, SYM><<<(unsigned)(tiles * best), NT, Sh::bytes, s>>>(a);
    return check_cuda(cudaGetLastError(), "gsf mma launch");
  }
}

// Symmetric half (SYM, p >= 3): only the J0 >= I0 values are computed and the rest mirrored, so
// the launch must write every row its elements touch (sym_covers); IGA_GSF_SYM=0 selects the
// full computation (A/B).
template <int P, int Q>
struct Launch {
  static int run(const GsfArgs& a, cudaStream_t s) {
    static const bool no_sym = [] {
      const char* e = getenv("IGA_GSF_SYM");
      return e != nullptr && e[0] == '0' && e[1] == 0;
    }();
    // p <= 2: the ring and run-emission work outweighs the halved stages B and S
    // (tools/tile_shapes.py, IGA_GSF_TILE=0: 64^3 p = 2 stiffness 0.430 vs 0.422 ms, p = 1 mass
    // 0.197 vs 0.123); C4 (p = 4): 10.19 vs 11.71 ms
    const bool sym = sym_covers(a, P) && !no_sym && P >= 3;
    if (sym) {
      const int rc = sym_prezero(a, P, s);
      if (rc != IGA_OK) return rc;
    }
    if (a.op == IGA_OP_MASS) return sym ? launch_t<P, Q, false, true>(a, s) : launch_t<P, Q, false>(a, s);
    if constexpr (P >= 1) return sym ? launch_t<P, Q, true, true>(a, s) : launch_t<P, Q, true>(a, s);
    set_error("derivatives require degree >= 1");
    return IGA_EINVAL;
  }
};

}  // namespace mma

int launch_gsf_mma(const GsfArgs& a, int p, int q, cudaStream_t s) {
  return dispatch_pq<mma::Launch>(p, q, a, s);
}

}  // namespace iga

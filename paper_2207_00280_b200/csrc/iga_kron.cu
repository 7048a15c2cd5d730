// Separable integration + assembly (IGA_METHOD_SEPARABLE) for a scalar
// coefficient on the tensor-product mesh with the identity geometry map.
//
// With W(k0,k1,k2) = c jac w_k0 w_k1 w_k2 the element quadrature of the reference
// (integrators.py:77-151) factorises exactly per axis, and so does its sum over the
// elements supporting a pair (assembly.py:80-82):
//
//   M[I,J] = c jac  m(I0,J0) m(I1,J1) m(I2,J2)
//   S[I,J] = c jac (k0 m1 m2 + m0 k1 m2 + m0 m1 k2)
//   m(I,J) = sum_e sum_q w_q V_e(I-e,q) V_e(J-e,q),   k: same with derivatives D
//
// i.e. the global matrix is a sum of Kronecker products of assembled 1D band
// matrices -- sum factorisation carried to its limit for a rank-one weight tensor.
// The 1D matrices are integrated by Gauss quadrature inside the kernel (per CTA,
// into shared memory); every CSR value then costs a multiply and an FMA on two
// per-pencil factors, so the kernel is bound by the HBM write of the CSR values.
// The element slab [el_begin, el_end) (multi-GPU) restricts only the axis-0 factor.
//
// One CTA per (I0, I1) row pencil (grid-stride): the pencil's rows I2 = 0..N-1 are
// contiguous in the CSR; they are produced in shared memory a few rows at a time
// and written by TMA bulk stores.
#include "iga_args.cuh"
#include "iga_band.cuh"
#include "iga_dispatch.cuh"

namespace iga {

#ifndef KRON_MINB
#define KRON_MINB 2
#endif

// high degrees (p >= 6): every row is split into KRON_HS halves by pair range, each half
// its own chunk, so a chunk is ~27 KB and two 512-thread CTAs fit one SM (one CTA's per-row
// barrier overlaps the other's work)
#ifndef KRON_HS
#define KRON_HS 2
#endif
__host__ __device__ constexpr int kron_split(int P) { return P >= 6 ? KRON_HS : 1; }
// threads per CTA: one per value of an interior row (NB^3, rounded to warps, <= 1024); 512
// for the split rows of the high degrees
__host__ __device__ constexpr int kron_nt(int P) {
  return kron_split(P) > 1 ? 512
         : ((2 * P + 1) * (2 * P + 1) * (2 * P + 1) + 31) / 32 * 32 > 1024
             ? 1024
             : ((2 * P + 1) * (2 * P + 1) * (2 * P + 1) + 31) / 32 * 32;
}
// resident CTAs per SM asked of the register allocator
__host__ __device__ constexpr int kron_minb(int P) {
  return kron_split(P) > 1 ? 2 : (P > 3 || kron_nt(P) * KRON_MINB > 1536 ? 1 : KRON_MINB);
}
// rows per staged chunk (one TMA bulk store each)
// (measured on B200: 16 rows with 2 CTAs/SM for the small meshes, where the chunk
// count per pencil is low; 8 rows for K > 96)
#ifndef KRON_GS
#define KRON_GS 16
#endif
__host__ __device__ constexpr int kron_rows(int P, bool small_mesh) {
  // high degrees: one row (NB^3 = 2197..6859 values) per staged chunk
  return P <= 2 ? 16 : (P == 3 ? (small_mesh ? KRON_GS : 8) : (P <= 5 ? 4 : 1));
}
#ifndef KRON_NBUF
#define KRON_NBUF 2
#endif
// staging buffers per CTA (2: one bulk store in flight while the next chunk is produced;
// 3 and 4 with proportionally fewer rows per chunk measured slower)
// high degrees stage one row per chunk: three buffers keep two bulk stores in flight
__host__ __device__ constexpr int kron_nbuf(int P) { return P <= 5 ? KRON_NBUF : 3; }
// doubles per staging buffer: a chunk of full rows plus 16-byte alignment padding
__host__ __device__ constexpr int kron_stage(int P, int G) {
  // (a split row: the values of its larger half)
  return (G * (((2 * P + 1) * (2 * P + 1) + kron_split(P) - 1) / kron_split(P)) * (2 * P + 1) + 3) / 2 * 2;
}

__device__ __forceinline__ void bulk_store(double* g, const double* sm, int bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(g),
               "r"((unsigned)__cvta_generic_to_shared(sm)), "r"(bytes)
               : "memory");
}

// CSR values are produced into a shared-memory chunk laid out exactly like its
// global range (same address mod 16) and leave with one TMA bulk store per chunk:
// the copy engine writes whole lines whatever the row alignment (rows of NB^3
// doubles are not 128-byte multiples; per-thread stores of them straddle lines and
// ran at half the write bandwidth), and the store issue leaves the SM pipes.
template <int P, int Q, int G>
__global__ void __launch_bounds__(kron_nt(P), kron_minb(P)) k_kron3(KronArgs a) {
  constexpr int NB = 2 * P + 1;
  constexpr int NT = kron_nt(P);
  constexpr int HS = kron_split(P);
  static_assert(HS == 1 || G == 1, "split rows are one-row chunks");
  constexpr int HP0 = (NB * NB + HS - 1) / HS;        // pairs of a full half
  constexpr int NE = (HP0 * NB + NT - 1) / NT;        // interior values per thread and (half) row
  constexpr int SG = kron_stage(P, G);
  extern __shared__ __align__(16) double2 tb[];  // [2][N][NB] (m, k): all elements, slab
  __shared__ double w[Q];
  const int K = a.K, tid = threadIdx.x;
  const int64_t N = (int64_t)K + P;
  const bool stiff = a.op != IGA_OP_MASS;
  // axis 0 sees only the slab's elements [el_begin, el_end); its table is a copy of the
  // full one unless the slab is a proper subset
  const bool full = a.el_begin <= 0 && a.el_end >= K;
  const double2* tb0 = full ? tb : tb + N * NB;
  // [NBUF][SG] (after both tables even when the slab table is unused: the larger
  // footprint measured ~4% faster on B200 than packing the staging after one table)
  double* stage = reinterpret_cast<double*>(tb + 2 * N * NB);
#ifdef KRON_EMPTY
  if (a.K > 0) return;
#endif
  // Work: chunks of G rows of a pencil, in CSR order; CTA b takes the contiguous
  // range [b U / grid, (b+1) U / grid) of the U chunks (balanced to a chunk)
  const int nch = (int)((N + G - 1) / G);
  // units: (pencil, half, chunk), in that order
  const int64_t nunit = (int64_t)(a.plane_end - a.plane_begin) * N * HS * nch;
  const int64_t u_lo0 = nunit * blockIdx.x / gridDim.x, u_hi0 = nunit * (blockIdx.x + 1) / gridDim.x;
  if (a.band) {
    // 1D band matrices precomputed once per step (iga_band_tables): a short copy instead
    // of the quadrature in every CTA; the axis-0 rows of an element slab are integrated
    // here for the CTA's planes only
    for (int u = tid; u < N * NB; u += NT) tb[u] = __ldg(a.band + u);
    if (!full) {
      if (tid < Q) w[tid] = a.weights[tid];
      __syncthreads();
      const int i0lo = a.plane_begin + (int)(u_lo0 / nch / HS / N);
      const int i0hi = a.plane_begin + (int)((u_hi0 - 1) / nch / HS / N);
      for (int u = tid; u < (i0hi - i0lo + 1) * NB; u += NT) {
        const int I0 = i0lo + u / NB, d = u % NB;
        tb[N * NB + I0 * NB + d] =
            band1d_el<P, Q>(a.V, a.D, K, w, I0, d, a.el_begin, a.el_end, stiff, a.wt);
      }
    }
    __syncthreads();
  } else {
    build_band_tables<P, Q>(a.V, a.D, a.weights, K, stiff, a.el_begin, a.el_end, !full, tb, stage,
                            kron_nbuf(P) * SG, w, tid, NT, a.wt);
  }

#ifdef KRON_PROLOGUE_ONLY
  if (a.K > 0) return;
#endif
  int chunk = 0;  // chunks issued by this CTA (selects the staging buffer)
  const int64_t T = band_prefix(N, P, N);  // values of a full-length band row set
  // the chunk produced last, stored after the next barrier (thread 0)
  double* pg = nullptr;
  const double* psb = nullptr;
  int plen = 0, ppad = 0;
  auto issue = [&]() {
    if (pg == nullptr) return;
    // 16-byte aligned middle by TMA; an unaligned first / last value by plain stores
    int n = plen - ppad;
    if (ppad) pg[0] = psb[0];
    if (n & 1) { pg[plen - 1] = psb[plen - 1]; --n; }
    if (n > 0) bulk_store(pg + ppad, psb + ppad, n * 8);
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    pg = nullptr;
  };
  const int64_t u_lo = u_lo0, u_hi = u_hi0;
  double* vals = nullptr;  // first value of the current pencil
  for (int64_t ph = u_lo / nch; ph * nch < u_hi; ++ph) {
    const int64_t pen = ph / HS;
    const int half = (int)(ph - pen * HS);
    const int I0 = a.plane_begin + (int)(pen / N), I1 = (int)(pen % N);
    // consecutive pencils are contiguous in the CSR: one 64-bit rowptr per CTA
    if (vals == nullptr) vals = a.values + (rowptr3(I0, I1, 0, P, N) - a.base);
    const double2* r0 = tb0 + I0 * NB;
    const int lod0 = max(0, P - I0), lod1 = max(0, P - I1);
    const int c0 = (int)band_cnt(I0, P, N), c1 = (int)band_cnt(I1, P, N), c01 = c0 * c1;
    const double2* r1 = tb + I1 * NB;
    // this half's pairs [b0, b0 + nb) (the whole row when HS = 1)
    const int hp = (c01 + HS - 1) / HS, b0 = half * hp, nb = min(c01, b0 + hp) - b0;
    // per-pair factors: value = fa * m2 + fb * k2
    const unsigned inv1 = (1u << 20) / (unsigned)c1 + 1u;  // b / c1 for b < 2^20 / NB
    auto factors = [&](int b, double& fa, double& fb) {
      const int bq = (int)(((unsigned)b * inv1) >> 20);
      const double2 x0 = r0[lod0 + bq], x1 = r1[lod1 + b - bq * c1];
      const double mm = a.jc * (x0.x * x1.x);
      if (a.op == IGA_OP_MASS) {
        fa = mm; fb = 0.0;
      } else {
        double s = a.jc * (x0.y * x1.x + x0.x * x1.y);
        if (a.op == IGA_OP_STIFFNESS_MASS) s += mm;
        fa = s; fb = mm;
      }
    };
    const int ncnt = c01 * NB;   // values of an interior row
    const int hcnt = nb * NB;    // values of this half of an interior row
    double fa[NE], fb[NE];
    int d2[NE], bp[NE];  // the thread's (pair b - b0, band offset d2) per slot j of the half row
#pragma unroll
    for (int j = 0; j < NE; ++j) {
      const int e = tid + j * NT;  // value index inside the half row
      fa[j] = fb[j] = 0.0;
      d2[j] = e % NB;
      bp[j] = e / NB;
      if (e < hcnt) factors(b0 + bp[j], fa[j], fb[j]);
    }
    const int64_t pc0 = u_lo - ph * nch, pc1 = u_hi - ph * nch;
    const int ch0 = pc0 > 0 ? (int)pc0 : 0, ch1 = pc1 < nch ? (int)pc1 : nch;
    // value offset of row R0 inside the pencil (int: a pencil holds < 2^31 values);
    // full-band chunks advance it without the band_prefix arithmetic
    int off0 = c01 * (int)band_prefix(ch0 * G, P, N);
    for (int R0 = ch0 * G; R0 < ch1 * G; R0 += G, ++chunk) {
      const int R1 = min((int)N, R0 + G);
      const bool fast = R0 >= P && R0 + G <= K;
      // rows of the chunk: their band counts sum (one row: band_cnt, no band_prefix pair)
      const int rows_c2 = fast ? G * NB
                               : (G == 1 ? (int)band_cnt(R0, P, N)
                                         : (int)(band_prefix(R1, P, N) - band_prefix(R0, P, N)));
      const int len = nb * rows_c2;                       // values of this chunk
      double* g = vals + off0 + (HS > 1 ? b0 * rows_c2 : 0);  // (HS > 1: one row)
      off0 += c01 * rows_c2;
      const int pad = (int)((reinterpret_cast<uintptr_t>(g) >> 3) & 1);
      double* buf = stage + (chunk % kron_nbuf(P)) * SG;
      // One CTA barrier per chunk: before it, the bulk store that last read this buffer
      // (chunk - NBUF, issued at the top of chunk - NBUF + 1) has finished reading it;
      // after it, the previous chunk is complete in shared memory and leaves.
      if (tid == 0) asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(kron_nbuf(P) - 2) : "memory");
      __syncthreads();
      if (tid == 0) issue();
      double* sb = buf + pad;
      // truncated-band rows (I2 < P or I2 >= K): a row holds the same (pair b, offset d2)
      // values as an interior row for d2 in [lod2, lod2 + c2), at b c2 + d2 - lod2, so every
      // thread reuses its interior slots' factors (one multiply-add per value; the per-value
      // division and pair-factor table of round 1 made these rows ~2.5x dearer per value)
      auto boundary_row = [&](int I2, int loc) {
        const double2* t2 = tb + I2 * NB;
        const int c2 = (int)band_cnt(I2, P, N), lod2 = max(0, P - I2);
#pragma unroll
        for (int j = 0; j < NE; ++j) {
          const int e = tid + j * NT;
          if (e < hcnt && d2[j] >= lod2 && d2[j] < lod2 + c2) {
            const double2 x2 = t2[d2[j]];
            sb[loc + bp[j] * c2 + d2[j] - lod2] = fa[j] * x2.x + fb[j] * x2.y;
          }
        }
        return loc + nb * c2;
      };
      int loc = 0;  // value offset of the next row inside the chunk
      for (int I2 = R0; I2 < min(R1, P); ++I2) loc = boundary_row(I2, loc);
      // full-band rows [max(R0,P), min(R1,K)): a fixed (pair, d2) per thread, rows hcnt apart
      const int ib = max(R0, P), nr = min(R1, K) - ib;
      if (nr > 0) {
        const double2* t2 = tb + ib * NB;
        double* sbi = sb + loc;
#pragma unroll
        for (int r = 0; r < G; ++r)
          if (r < nr) {
#pragma unroll
            for (int j = 0; j < NE; ++j) {
              const int e = tid + j * NT;
              if (e < hcnt) {
                const double2 x2 = t2[r * NB + d2[j]];
                sbi[r * hcnt + e] = fa[j] * x2.x + fb[j] * x2.y;
              }
            }
          }
        loc += nr * hcnt;
      }
      for (int I2 = max(R0, max(K, P)); I2 < R1; ++I2) loc = boundary_row(I2, loc);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      if (tid == 0) {
        pg = g; psb = sb; plen = len; ppad = pad;
      }
    }
    (void)ncnt;
    if (half == HS - 1) vals += (int64_t)c01 * T;
  }
  __syncthreads();
  if (tid == 0) {
    issue();
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}

// K1 + the band matrices, one CTA per RB band rows: each CTA evaluates the Cox-de Boor
// tables of the elements its rows touch (its own and P halo elements, k_mesh_tables'
// arithmetic; halo elements are evaluated twice with identical bits), their element
// integrals, and the sums per band entry in build_band_tables' order -- so k_kron3
// produces the same bits either way, and the launch is a few latency rounds on several
// SMs instead of the quadrature prologue of every k_kron3 CTA.
// band rows per CTA (8; 2 for the high degrees, whose element tables fill static smem)
__host__ __device__ constexpr int band_rows(int P) { return P <= 5 ? 8 : 2; }
template <int P, int Q>
__global__ void __launch_bounds__(128) k_mesh_band(int K, const double* __restrict__ ref,
                                                   const double* __restrict__ weights, int stiff,
                                                   double* __restrict__ V, double* __restrict__ D,
                                                   double2* __restrict__ band,
                                                   const double* __restrict__ knots,
                                                   double* __restrict__ wt) {
  constexpr int kBandRows = band_rows(P);
  constexpr int M = P + 1, NB = 2 * P + 1, NEL = kBandRows + P;
  __shared__ double Vs[NEL * M * Q], Ds[NEL * M * Q];
  __shared__ double2 em[NEL * M * M];
  __shared__ double w[Q], wes[NEL * Q];  // reference weights; per-element weights (knots)
  const int N = K + P, tid = threadIdx.x, nt = blockDim.x;
  const int i_lo = blockIdx.x * kBandRows, i_hi = min(N, i_lo + kBandRows);
  const int e0 = max(0, i_lo - P), e1 = min(K, i_hi), ne = e1 - e0;
  if (tid < Q) w[tid] = weights[tid];
  if (knots) {  // w_k h_e / 2 of the CTA's elements (written once to wt by the CTA owning e)
    for (int u = tid; u < ne * Q; u += nt) {
      const int le = u / Q, k = u - le * Q, e = e0 + le;
      const double h = sub(__ldg(knots + P + e + 1), __ldg(knots + P + e));
      wes[u] = mul(weights[k], dvd(h, 2.0));
      if (wt && e >= i_lo) wt[e * Q + k] = wes[u];
    }
  }
  for (int u = tid; u < ne * Q; u += nt) {
    const int le = u / Q, k = u - le * Q, e = e0 + le;
    double vals[M], ders[M];
    cox_de_boor<P>(e, map_node(e, ref[k], K, P, knots), K, vals, stiff ? ders : nullptr, knots);
#pragma unroll
    for (int r = 0; r < M; ++r) {
      const int o = (le * M + r) * Q + k, og = (e * M + r) * Q + k;
      Vs[o] = vals[r];
      if (V) V[og] = vals[r];
      if (stiff) {
        Ds[o] = ders[r];
        if (D) D[og] = ders[r];
      }
    }
  }
  __syncthreads();
  for (int u = tid; u < ne * M * M; u += nt) {
    const int le = u / (M * M), r = (u / M) % M, c = u % M;
    const double* vr = Vs + (le * M + r) * Q;
    const double* vc = Vs + (le * M + c) * Q;
    double m = 0.0, k = 0.0;
    const double* we = knots ? wes + le * Q : w;
#pragma unroll
    for (int q = 0; q < Q; ++q) m += (we[q] * vr[q]) * vc[q];
    if (stiff) {
      const double* dr = Ds + (le * M + r) * Q;
      const double* dc = Ds + (le * M + c) * Q;
#pragma unroll
      for (int q = 0; q < Q; ++q) k += (we[q] * dr[q]) * dc[q];
    }
    em[u] = make_double2(m, k);
  }
  __syncthreads();
  for (int u = tid; u < (i_hi - i_lo) * NB; u += nt) {
    const int I = i_lo + u / NB, J = I + u % NB - P;
    const int lo = max(max(I, J) - P, 0), hi = min(min(I, J) + 1, K);
    double m = 0.0, k = 0.0;
    for (int e = lo; e < hi; ++e) {
      const double2 x = em[((e - e0) * M + I - e) * M + J - e];
      m += x.x;
      k += x.y;
    }
    band[I * NB + u % NB] = make_double2(m, k);
  }
}

template <int P, int Q>
struct BandLaunch {
  static int run(int K, const double* ref, const double* weights, int stiff, double* V, double* D,
                 double2* band, const double* knots, double* wt, cudaStream_t s) {
    const int N = K + P;
    k_mesh_band<P, Q><<<(N + band_rows(P) - 1) / band_rows(P), 128, 0, s>>>(
        K, ref, weights, stiff, V, D, band, knots, wt);
    return check_cuda(cudaGetLastError(), "band launch");
  }
};

int launch_band_tables(int K, int p, int q, const double* ref, const double* weights, int stiff,
                       double* V, double* D, double* band, const double* knots, double* wt,
                       cudaStream_t s) {
  return dispatch_pq_all<BandLaunch>(p, q, K, ref, weights, stiff, V, D,
                                     reinterpret_cast<double2*>(band), knots, wt, s);
}

template <int P, int Q, int G>
static int launch_kron_g(const KronArgs& a, cudaStream_t s) {
  const int64_t N = (int64_t)a.K + P;
  constexpr int NT = kron_nt(P);
  const size_t smem = 2 * sizeof(double2) * N * (2 * P + 1) + kron_nbuf(P) * sizeof(double) * kron_stage(P, G);
  if (smem > 220 * 1024) {
    set_error("separable path: 1D band tables of K=%d do not fit shared memory", a.K);
    return IGA_EUNSUPPORTED;
  }
  const void* fn = reinterpret_cast<const void*>(k_kron3<P, Q, G>);
  cudaError_t e = smem_attr_once(fn, smem, true);
  if (e != cudaSuccess) return check_cuda(e, "kron smem attr");
  const int per_sm = blocks_per_sm_once(fn, NT, smem), sms = sm_count();
  const int64_t nunit = (int64_t)(a.plane_end - a.plane_begin) * N * kron_split(P) * ((N + G - 1) / G);
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > nunit) grid = nunit;
  if (grid <= 0) return IGA_OK;
  k_kron3<P, Q, G><<<(unsigned)grid, NT, smem, s>>>(a);
  return check_cuda(cudaGetLastError(), "kron launch");
}

template <int P, int Q>
struct KronLaunch {
  static int run(const KronArgs& a, cudaStream_t s) {
    constexpr int Gs = kron_rows(P, true), Gl = kron_rows(P, false);
    if (Gs != Gl && a.K <= 96) return launch_kron_g<P, Q, Gs>(a, s);
    return launch_kron_g<P, Q, Gl>(a, s);
  }
};

int launch_kron(const KronArgs& a, int p, int q, cudaStream_t s) {
  return dispatch_pq_all<KronLaunch>(p, q, a, s);
}

}  // namespace iga

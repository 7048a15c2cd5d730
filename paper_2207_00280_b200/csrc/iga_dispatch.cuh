// Compile-time dispatch over the supported (p, q) grid.
//
//   every kernel family:        0 <= p <= kMaxPLow (5), 1 <= q <= min(p + 3, 8)
//   high degrees (opt-in):      6 <= p <= kMaxP (9),    q in {p + 1, p + 2}, q <= kMaxQ (10)
//
// L<P, Q>::run(args...) is instantiated only for supported pairs; anything else
// returns IGA_EUNSUPPORTED with a message (-> ValueError in Python).  Families whose
// kernels serve the high degrees (the paper's p = 9 Gram) use the
// *_all variants; the others keep the low grid and report which paths cover high p.
#pragma once

#include <utility>

#include "iga_common.cuh"

namespace iga {

constexpr int kMaxPLow = 5;   // every kernel family
constexpr int kMaxQLow = 8;

template <int P, int Q>
constexpr bool supported_pq() {
  if (P <= kMaxPLow) return Q >= 1 && Q <= P + 3 && Q <= kMaxQLow;
  return P <= kMaxP && (Q == P + 1 || Q == P + 2) && Q <= kMaxQ;
}

template <template <int, int> class L, int P, int Q, bool HI, typename... A>
int run_if_supported(A&&... a) {
  if constexpr (supported_pq<P, Q>() && (HI || P <= kMaxPLow)) {
    return L<P, Q>::run(std::forward<A>(a)...);
  } else if constexpr (P > kMaxPLow && !HI) {
    set_error("degree p=%d: this path runs p <= %d; for p <= %d use the separable (scalar "
              "coefficient) or classical method, or element-local sum factorization",
              P, kMaxPLow, kMaxP);
    return IGA_EUNSUPPORTED;
  } else {
    set_error("quadrature points q=%d not supported on device for p=%d (p <= 5: 1 <= q <= p+3, "
              "q <= 8; 6 <= p <= 9: q = p+1 or p+2, q <= 10)", Q, P);
    return IGA_EUNSUPPORTED;
  }
}

template <template <int, int> class L, int P, bool HI, typename... A>
int dispatch_q(int q, A&&... a) {
  switch (q) {
    case 1: return run_if_supported<L, P, 1, HI>(std::forward<A>(a)...);
    case 2: return run_if_supported<L, P, 2, HI>(std::forward<A>(a)...);
    case 3: return run_if_supported<L, P, 3, HI>(std::forward<A>(a)...);
    case 4: return run_if_supported<L, P, 4, HI>(std::forward<A>(a)...);
    case 5: return run_if_supported<L, P, 5, HI>(std::forward<A>(a)...);
    case 6: return run_if_supported<L, P, 6, HI>(std::forward<A>(a)...);
    case 7: return run_if_supported<L, P, 7, HI>(std::forward<A>(a)...);
    case 8: return run_if_supported<L, P, 8, HI>(std::forward<A>(a)...);
    case 9: return run_if_supported<L, P, 9, HI>(std::forward<A>(a)...);
    case 10: return run_if_supported<L, P, 10, HI>(std::forward<A>(a)...);
    default:
      set_error("quadrature points q=%d not supported on device (1..%d)", q, kMaxQ);
      return IGA_EUNSUPPORTED;
  }
}

template <template <int, int> class L, bool HI, typename... A>
int dispatch_pq_impl(int p, int q, A&&... a) {
  switch (p) {
    case 0: return dispatch_q<L, 0, HI>(q, std::forward<A>(a)...);
    case 1: return dispatch_q<L, 1, HI>(q, std::forward<A>(a)...);
    case 2: return dispatch_q<L, 2, HI>(q, std::forward<A>(a)...);
    case 3: return dispatch_q<L, 3, HI>(q, std::forward<A>(a)...);
    case 4: return dispatch_q<L, 4, HI>(q, std::forward<A>(a)...);
    case 5: return dispatch_q<L, 5, HI>(q, std::forward<A>(a)...);
    case 6: return dispatch_q<L, 6, HI>(q, std::forward<A>(a)...);
    case 7: return dispatch_q<L, 7, HI>(q, std::forward<A>(a)...);
    case 8: return dispatch_q<L, 8, HI>(q, std::forward<A>(a)...);
    case 9: return dispatch_q<L, 9, HI>(q, std::forward<A>(a)...);
    default:
      set_error("degree p=%d not supported on device (0..%d)", p, kMaxP);
      return IGA_EUNSUPPORTED;
  }
}

// low grid only (p <= 5)
template <template <int, int> class L, typename... A>
int dispatch_pq(int p, int q, A&&... a) {
  return dispatch_pq_impl<L, false>(p, q, std::forward<A>(a)...);
}
// low grid + high degrees (p <= 9)
template <template <int, int> class L, typename... A>
int dispatch_pq_all(int p, int q, A&&... a) {
  return dispatch_pq_impl<L, true>(p, q, std::forward<A>(a)...);
}

template <template <int> class L, bool HI, typename... A>
int dispatch_p_impl(int p, A&&... a) {
  switch (p) {
    case 0: return L<0>::run(std::forward<A>(a)...);
    case 1: return L<1>::run(std::forward<A>(a)...);
    case 2: return L<2>::run(std::forward<A>(a)...);
    case 3: return L<3>::run(std::forward<A>(a)...);
    case 4: return L<4>::run(std::forward<A>(a)...);
    case 5: return L<5>::run(std::forward<A>(a)...);
    default:
      if constexpr (HI) {
        switch (p) {
          case 6: return L<6>::run(std::forward<A>(a)...);
          case 7: return L<7>::run(std::forward<A>(a)...);
          case 8: return L<8>::run(std::forward<A>(a)...);
          case 9: return L<9>::run(std::forward<A>(a)...);
          default: break;
        }
      }
      set_error("degree p=%d not supported on device (0..%d)", p, HI ? kMaxP : kMaxPLow);
      return IGA_EUNSUPPORTED;
  }
}

template <template <int> class L, typename... A>
int dispatch_p(int p, A&&... a) {
  return dispatch_p_impl<L, false>(p, std::forward<A>(a)...);
}
template <template <int> class L, typename... A>
int dispatch_p_all(int p, A&&... a) {
  return dispatch_p_impl<L, true>(p, std::forward<A>(a)...);
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace iga

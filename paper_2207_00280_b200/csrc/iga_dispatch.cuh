// Compile-time dispatch over the supported (p, q) grid:
//   0 <= p <= kMaxP, 1 <= q <= min(p + 3, kMaxQ).
// L<P, Q>::run(args...) is instantiated only for supported pairs; anything
// else returns IGA_EUNSUPPORTED with a message (-> ValueError in Python).
#pragma once

#include <utility>

#include "iga_common.cuh"

namespace iga {

template <template <int, int> class L, int P, int Q, typename... A>
int run_if_supported(A&&... a) {
  if constexpr (Q >= 1 && Q <= P + 3 && Q <= kMaxQ) {
    return L<P, Q>::run(std::forward<A>(a)...);
  } else {
    set_error("quadrature points q=%d not supported on device for p=%d (need 1 <= q <= p+3)", Q, P);
    return IGA_EUNSUPPORTED;
  }
}

template <template <int, int> class L, int P, typename... A>
int dispatch_q(int q, A&&... a) {
  switch (q) {
    case 1: return run_if_supported<L, P, 1>(std::forward<A>(a)...);
    case 2: return run_if_supported<L, P, 2>(std::forward<A>(a)...);
    case 3: return run_if_supported<L, P, 3>(std::forward<A>(a)...);
    case 4: return run_if_supported<L, P, 4>(std::forward<A>(a)...);
    case 5: return run_if_supported<L, P, 5>(std::forward<A>(a)...);
    case 6: return run_if_supported<L, P, 6>(std::forward<A>(a)...);
    case 7: return run_if_supported<L, P, 7>(std::forward<A>(a)...);
    case 8: return run_if_supported<L, P, 8>(std::forward<A>(a)...);
    default:
      set_error("quadrature points q=%d not supported on device (1..%d)", q, kMaxQ);
      return IGA_EUNSUPPORTED;
  }
}

template <template <int, int> class L, typename... A>
int dispatch_pq(int p, int q, A&&... a) {
  switch (p) {
    case 0: return dispatch_q<L, 0>(q, std::forward<A>(a)...);
    case 1: return dispatch_q<L, 1>(q, std::forward<A>(a)...);
    case 2: return dispatch_q<L, 2>(q, std::forward<A>(a)...);
    case 3: return dispatch_q<L, 3>(q, std::forward<A>(a)...);
    case 4: return dispatch_q<L, 4>(q, std::forward<A>(a)...);
    case 5: return dispatch_q<L, 5>(q, std::forward<A>(a)...);
    default:
      set_error("degree p=%d not supported on device (0..%d)", p, kMaxP);
      return IGA_EUNSUPPORTED;
  }
}

template <template <int> class L, typename... A>
int dispatch_p(int p, A&&... a) {
  switch (p) {
    case 0: return L<0>::run(std::forward<A>(a)...);
    case 1: return L<1>::run(std::forward<A>(a)...);
    case 2: return L<2>::run(std::forward<A>(a)...);
    case 3: return L<3>::run(std::forward<A>(a)...);
    case 4: return L<4>::run(std::forward<A>(a)...);
    case 5: return L<5>::run(std::forward<A>(a)...);
    default:
      set_error("degree p=%d not supported on device (0..%d)", p, kMaxP);
      return IGA_EUNSUPPORTED;
  }
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace iga

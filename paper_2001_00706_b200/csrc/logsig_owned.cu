// logsig_owned.cu -- instances of the compile-time K5 (logsig_owned.cuh) and their lookup.
#include <utility>
#include "logsig_owned.cuh"

namespace sigb200 {
namespace {

constexpr size_t kOwnedMaxSmem = 227 * 1024 - 512;

template <int C, int N>
constexpr LogsigBwdLaunch entry() {
    if constexpr ((size_t)LT<C, N>::TOTAL * sizeof(float) <= kOwnedMaxSmem) return &launch_logsig_bwd_owned_t<C, N>;
    else return nullptr;
}

template <int C, int... Ns>
LogsigBwdLaunch pick(int N, std::integer_sequence<int, Ns...>) {
    LogsigBwdLaunch r = nullptr;
    ((N == Ns + 1 ? (r = entry<C, Ns + 1>(), 0) : 0), ...);
    return r;
}

template <int C, int N>
constexpr LogsigFwdLaunch fentry() {
    if constexpr (LogFwdT<C, N>::HS * 16 + LogFwdT<C, N>::XSP * 4 <= kOwnedMaxSmem) return &launch_logsig_fwd_t<C, N>;
    else return nullptr;
}

template <int C, int... Ns>
LogsigFwdLaunch fpick(int N, std::integer_sequence<int, Ns...>) {
    LogsigFwdLaunch r = nullptr;
    ((N == Ns + 1 ? (r = fentry<C, Ns + 1>(), 0) : 0), ...);
    return r;
}

}  // namespace

LogsigFwdLaunch find_logsig_fwd_t(int C, int N) {
    switch (C) {
        case 1: return fpick<1>(N, std::make_integer_sequence<int, 12>{});
        case 2: return fpick<2>(N, std::make_integer_sequence<int, 12>{});
        case 4: return fpick<4>(N, std::make_integer_sequence<int, 7>{});
        case 8: return fpick<8>(N, std::make_integer_sequence<int, 5>{});
        default: return nullptr;
    }
}

namespace {
template <int C, int... Ns>
size_t fsmem(int N, int w, bool br, std::integer_sequence<int, Ns...>) {
    size_t r = 0;
    ((N == Ns + 1 ? (r = LogFwdT<C, Ns + 1>::smem(w, br), 0) : 0), ...);
    return r;
}
}  // namespace

size_t logsig_fwd_t_smem(int C, int N, int w, bool brackets) {
    switch (C) {
        case 1: return fsmem<1>(N, w, brackets, std::make_integer_sequence<int, 12>{});
        case 2: return fsmem<2>(N, w, brackets, std::make_integer_sequence<int, 12>{});
        case 4: return fsmem<4>(N, w, brackets, std::make_integer_sequence<int, 7>{});
        case 8: return fsmem<8>(N, w, brackets, std::make_integer_sequence<int, 5>{});
        default: return 0;
    }
}

LogsigBwdLaunch find_logsig_bwd_owned(int C, int N) {
    switch (C) {
        case 1: return pick<1>(N, std::make_integer_sequence<int, 12>{});
        case 2: return pick<2>(N, std::make_integer_sequence<int, 12>{});
        case 4: return pick<4>(N, std::make_integer_sequence<int, 7>{});
        case 8: return pick<8>(N, std::make_integer_sequence<int, 5>{});
        default: return nullptr;
    }
}

}  // namespace sigb200

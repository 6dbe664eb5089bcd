// sig_table.h -- dispatch table entries produced by gen_instances.py (one per supported (C, N)).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sigb200 {

struct FwdParams;
struct BwdParams;
struct GroupParams;
struct ScanParams;

using FwdLaunch = cudaError_t (*)(const FwdParams&, cudaStream_t);
using BwdLaunch = cudaError_t (*)(const BwdParams&, cudaStream_t);
using BwdSlots = int64_t (*)();
using FoldLaunch = cudaError_t (*)(const GroupParams&, unsigned ngroups, unsigned B, cudaStream_t);
using ScanLaunch = cudaError_t (*)(const ScanParams&, cudaStream_t);

struct KernelSet {
    int C, N;
    int pf0, pf1, pb;   // prefix lengths of the two forward variants and of the backward (-1: none)
    FwdLaunch fwd0, fwd1;
    BwdLaunch bwd;
    BwdSlots bwd_slots;         // CTAs of the (chunk-capable) backward resident per SM
    FoldLaunch fold;            // compiled ordered group fold (K3) for this (C, N)
    ScanLaunch scan;            // compiled blocked chunk scan (the time-parallel backward)
    bool fwd2;                  // fwd0 has the two-prefix forward (sig_fwd2_kernel, plain calls of B >= 64)
};

const KernelSet* kernels_c1(int N);
const KernelSet* kernels_c2(int N);
const KernelSet* kernels_c3(int N);
const KernelSet* kernels_c4(int N);
const KernelSet* kernels_c5(int N);
const KernelSet* kernels_c6(int N);
const KernelSet* kernels_c7(int N);
const KernelSet* kernels_c8(int N);

inline const KernelSet* find_kernels(int C, int N) {
    switch (C) {
        case 1: return kernels_c1(N);
        case 2: return kernels_c2(N);
        case 3: return kernels_c3(N);
        case 4: return kernels_c4(N);
        case 5: return kernels_c5(N);
        case 6: return kernels_c6(N);
        case 7: return kernels_c7(N);
        case 8: return kernels_c8(N);
        default: return nullptr;
    }
}

}  // namespace sigb200

// combine.cuh -- K3: the group-like product [x] on batches of signatures, sm_100a.
//
//   (A [x] B)_k = sum_{i=0}^{k} A_i (x) B_{k-i},  A_0 = B_0 = 1     (eq-tensorproduct)
//
// Used for signature_combine / multi_signature_combine and to fold the signatures
// of time chunks in order (Chen's identity eq-grouplike; "parallelised in the usual way
// for reductions").  One thread computes one output coefficient: word w at level k costs
// k-1 FMAs, A_i[w / C^(k-i)] * B_{k-i}[w mod C^(k-i)].  The work is small and HBM/L2-bound, so
// C and N are runtime values here (no template explosion).
//
// Group fold: a CTA loads G consecutive signatures of one path into shared memory and reduces
// them with an ordered binary tree (time order is preserved: [x] is associative but not
// commutative).  In-place update of the left operand is safe level by level, top-down: level k
// reads only levels < k of the left operand and its own coefficient.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sigb200 {

// 32-bit level tables (signatures here have S < 2^31 and C^N < 2^24)
struct TensorDims {
    int C, N, S;
    int off[18];     // off[k] = flat offset of level k (1-based), off[N+1] = S
    int pw[17];      // pw[k] = C^k
    uint32_t magic;  // n / C == __umulhi(n, magic) exactly for n < 2^32 / C
};

inline TensorDims make_dims(int C, int N) {
    TensorDims d{};
    d.C = C;
    d.N = N;
    d.pw[0] = 1;
    for (int k = 1; k <= 16; ++k) d.pw[k] = (k <= N + 1) ? d.pw[k - 1] * C : 0;
    d.off[1] = 0;
    for (int k = 1; k <= N; ++k) d.off[k + 1] = d.off[k] + d.pw[k];
    d.S = d.off[N + 1];
    d.magic = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)C - 1) / (uint64_t)C);
    return d;
}

__device__ __forceinline__ int level_of(const TensorDims& d, int f) {
    int k = 1;
    while (k < d.N && f >= d.off[k + 1]) ++k;
    return k;
}

// out = a [x] b for one flat coefficient (level k, word w): split w = u.v for |u| = i, i = k-1..1,
// peeling one letter at a time (no division other than by C, done with the magic multiplier)
__device__ __forceinline__ float mul_coef(const TensorDims& d, const float* a, const float* b, int k, int w) {
    float acc = a[d.off[k] + w] + b[d.off[k] + w];
    int u = w, v = 0, q = 1;
    for (int i = k - 1; i >= 1; --i) {
        const int u2 = (d.C == 1) ? u : (int)__umulhi((uint32_t)u, d.magic);
        v += (u - u2 * d.C) * q;
        q *= d.C;
        u = u2;
        acc = fmaf(a[d.off[i] + u], b[d.off[k - i] + v], acc);
    }
    return acc;
}

#ifdef SIG_DEFINE_COMBINE_KERNELS  // defined only by api.cu, the one TU that launches them
// ---------------------------------------------------------------- pairwise, batched
// row r: out + r*so = (a + r*sa) [x] (b + r*sb)
// Rows are grid-strided over gridDim.y (capped at 65535 by the launcher), so any row count works.
__global__ void combine_pair_kernel(const TensorDims d, const float* __restrict__ a, int64_t sa,
                                    const float* __restrict__ b, int64_t sb, float* __restrict__ out, int64_t so,
                                    int64_t rows) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= d.S) return;
    const int k = level_of(d, f);
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
        out[r * so + f] = mul_coef(d, a + r * sa, b + r * sb, k, f - d.off[k]);
}

// ---------------------------------------------------------------- VJP of a [x] b
//   ga_i[u] = go_i[u] + sum_{k>i} sum_v go_k[u v] b_{k-i}[v]
//   gb_j[v] = go_j[v] + sum_{k>j} sum_u go_k[u v] a_{k-j}[u]
// for one coefficient (level i, word u) of the row go; b / a nullptr = the identity
__device__ __forceinline__ float ga_coef(const TensorDims& d, const float* gor, const float* br, int i, int u) {
    float acc = gor[d.off[i] + u];
    if (!br) return acc;
    for (int k = i + 1; k <= d.N; ++k) {
        const int nv = d.pw[k - i];
        const float* gk = gor + d.off[k] + u * nv;
        const float* bk = br + d.off[k - i];
        for (int v = 0; v < nv; ++v) acc = fmaf(gk[v], bk[v], acc);
    }
    return acc;
}
__device__ __forceinline__ float gb_coef(const TensorDims& d, const float* gor, const float* ar, int j, int v) {
    float acc = gor[d.off[j] + v];
    if (!ar) return acc;
    for (int k = j + 1; k <= d.N; ++k) {
        const int nu = d.pw[k - j];
        const int stride = d.pw[j];
        const float* gk = gor + d.off[k] + v;
        const float* ak = ar + d.off[k - j];
        for (int uu = 0; uu < nu; ++uu) acc = fmaf(gk[uu * stride], ak[uu], acc);
    }
    return acc;
}

__global__ void combine_pair_bwd_kernel(const TensorDims d, const float* __restrict__ go, const float* __restrict__ a,
                                        const float* __restrict__ b, float* __restrict__ ga, float* __restrict__ gb,
                                        int64_t rows) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= d.S) return;
    const int i = level_of(d, f);
    const int u = f - d.off[i];
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
        const float* gor = go + r * d.S;
        if (ga) ga[r * d.S + f] = ga_coef(d, gor, b + r * d.S, i, u);
        if (gb) gb[r * d.S + f] = gb_coef(d, gor, a + r * d.S, i, u);
    }
}

// ---------------------------------------------------------------- Path interval queries
//   Sig(x_s .. x_{e-1}) = InvertSig(x_0 .. x_s) [x] Sig(x_0 .. x_{e-1}): with the
// stream rows sig[b, r] = Sig(x_0 .. x_{r+1}) and inv[b, r] = its inverse, query q = (s, e) reads
// inv row s-1 (the identity when s = 0) and sig row e-2.
struct PathQueryParams {
    TensorDims d;
    const float* sig;   // [B, M, S]
    const float* inv;   // [B, M, S]
    int64_t B, M, Q;
    const int64_t* qs;  // [Q] starts (device)
    const int64_t* qe;  // [Q] ends (device)
    float* out;         // [B, Q, S]
    // backward
    const float* gout;                       // [B, Q, S]
    const int* sig_ptr; const int* sig_q;    // CSR: sig row r -> the queries reading it (ascending)
    const int* inv_ptr; const int* inv_q;    // CSR: inv row r -> the queries reading it (ascending)
    float* gsig;                             // [B, M, S] overwritten
    float* ginv;                             // [B, M, S] overwritten
};

__global__ void path_query_kernel(const PathQueryParams p) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int S = p.d.S;
    if (e >= p.B * p.Q * S) return;
    const int64_t bq = e / S;
    const int f = (int)(e - bq * S);
    const int64_t b = bq / p.Q, q = bq - b * p.Q;
    const int64_t s0 = p.qs[q], e0 = p.qe[q];
    const float* sr = p.sig + ((size_t)b * p.M + (e0 - 2)) * S;
    if (s0 == 0) {
        p.out[e] = sr[f];
        return;
    }
    const float* ir = p.inv + ((size_t)b * p.M + (s0 - 1)) * S;
    const int k = level_of(p.d, f);
    p.out[e] = mul_coef(p.d, ir, sr, k, f - p.d.off[k]);
}

// dL/d(sig row r) = sum over the queries reading it of the b-side VJP, in ascending query order;
// dL/d(inv row r) likewise with the a-side VJP (deterministic: no atomics)
__global__ void path_query_bwd_kernel(const PathQueryParams p) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int S = p.d.S;
    if (e >= p.B * p.M * S) return;
    const int64_t br = e / S;
    const int f = (int)(e - br * S);
    const int64_t b = br / p.M, r = br - b * p.M;
    const int i = level_of(p.d, f);
    const int u = f - p.d.off[i];
    float acc = 0.0f;
    for (int t = p.sig_ptr[r]; t < p.sig_ptr[r + 1]; ++t) {
        const int q = p.sig_q[t];
        const int64_t s0 = p.qs[q];
        const float* ar = (s0 == 0) ? nullptr : p.inv + ((size_t)b * p.M + (s0 - 1)) * S;
        acc += gb_coef(p.d, p.gout + ((size_t)b * p.Q + q) * S, ar, i, u);
    }
    p.gsig[e] = acc;
    acc = 0.0f;
    for (int t = p.inv_ptr[r]; t < p.inv_ptr[r + 1]; ++t) {
        const int q = p.inv_q[t];
        const float* sr = p.sig + ((size_t)b * p.M + (p.qe[q] - 2)) * S;
        acc += ga_coef(p.d, p.gout + ((size_t)b * p.Q + q) * S, sr, i, u);
    }
    p.ginv[e] = acc;
}

// ---------------------------------------------------------------- time-parallel backward
// chunk signatures S_j of each path, j < m, laid out [B, m, S].
// One Hillis-Steele step of the inclusive ordered product along j (Chen's identity, eq-grouplike):
//   prefix:  out[b, j] = in[b, j - o] [x] in[b, j]   (j >= o, else a copy)
//   suffix:  out[b, j] = in[b, j] [x] in[b, j + o]   (j + o < m, else a copy)
__global__ void chunk_scan_step_kernel(const TensorDims d, const float* __restrict__ in, float* __restrict__ out,
                                       int64_t B, int64_t m, int64_t o, int suffix) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= B * m * d.S) return;
    const int64_t bj = e / d.S;
    const int f = (int)(e - bj * d.S);
    const int64_t j = bj % m;
    const float* row = in + bj * d.S;
    const int k = level_of(d, f);
    if (!suffix && j >= o) out[e] = mul_coef(d, in + (bj - o) * d.S, row, k, f - d.off[k]);
    else if (suffix && j + o < m) out[e] = mul_coef(d, row, in + (bj + o) * d.S, k, f - d.off[k]);
    else out[e] = row[f];
}

// gradient at the end of chunk j: Sig = P_{j+1} [x] Q_j with Q_j = S_{j+1} [x] .. [x] S_{m-1}
// (the inclusive suffix product at j + 1; the identity for the last chunk), so
// dL/dP_{j+1} = the a-side VJP of that product at gbar[b]
__global__ void chunk_gend_kernel(const TensorDims d, const float* __restrict__ gbar, const float* __restrict__ sfx,
                                  int64_t B, int64_t m, float* __restrict__ gend) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= B * m * d.S) return;
    const int64_t bj = e / d.S;
    const int f = (int)(e - bj * d.S);
    const int64_t b = bj / m, j = bj - b * m;
    const int i = level_of(d, f);
    gend[e] = ga_coef(d, gbar + b * d.S, (j + 1 < m) ? sfx + (bj + 1) * d.S : nullptr, i, f - d.off[i]);
}

// the first point of chunk j >= 1 is also the last point of chunk j - 1: add the share chunk j
// wrote to edge (runs after the chunk backward, in stream order -- deterministic)
__global__ void chunk_edge_fixup_kernel(float* __restrict__ grad_path, const float* __restrict__ edge, int64_t B,
                                        int64_t m, int64_t chunk_len, int64_t L, int has_bp, int C) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= B * (m - 1) * C) return;
    const int64_t bj = e / C;
    const int c = (int)(e - bj * C);
    const int64_t b = bj / (m - 1), j = 1 + (bj - b * (m - 1));
    const int64_t row = j * chunk_len - has_bp;  // augmented point j * chunk_len
    grad_path[(b * L + row) * C + c] += edge[(b * m + j) * C + c];
}

// ---------------------------------------------------------------- word reversal alpha
// alpha(x)[a_1 .. a_k] = x[a_k .. a_1] on every level: the anti-automorphism with
// alpha(A [x] B) = alpha(B) [x] alpha(A) and alpha(exp(z)) = exp(z), used for the inverse option
// (R18).  Row r of in (stride si) -> row r of out (stride so); in == out permutes in place
// (each pair {w, rev(w)} is swapped by the thread holding the smaller index).
__global__ void word_reverse_kernel(const TensorDims d, const float* in, int64_t si, float* out, int64_t so,
                                    int64_t rows) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rows * d.S) return;
    const int64_t r = e / d.S;
    const int f = (int)(e - r * d.S);
    const int k = level_of(d, f);
    int w = f - d.off[k], rev = 0;
    for (int q = 0; q < k; ++q) {
        const int w2 = (d.C == 1) ? w : (int)__umulhi((uint32_t)w, d.magic);
        rev = rev * d.C + (w - w2 * d.C);
        w = w2;
    }
    const int g = d.off[k] + rev;
    if (in == out) {
        if (g > f) {
            float* row = out + r * so;
            const float t = row[f];
            row[f] = row[g];
            row[g] = t;
        }
    } else {
        out[r * so + g] = in[r * si + f];
    }
}
#endif  // SIG_DEFINE_COMBINE_KERNELS

// ---------------------------------------------------------------- ordered group fold in smem
struct GroupParams {
    TensorDims d;
    const float* in;
    int64_t in_sj, in_sb;    // element (j, b) at in + j*in_sj + b*in_sb
    int64_t n;               // elements per path
    int G;                   // group size (power of two)
    float* out;
    int64_t out_sj, out_sb;  // group result (g, b) at out + g*out_sj + b*out_sb
    int64_t B;               // paths (grid-strided over gridDim.y, which is capped at 65535)
};

// blocked ordered scan along the chunk axis (scan_group_t_kernel, chunk_block_scan_kernel):
// elements in[b*m + j] (rows of S floats), groups of g, carries [B, ng]
struct ScanParams {
    const float* in;
    float* out;          // [B, m, S] or nullptr
    float* tot;          // [B, ng, S] group totals or nullptr
    const float* carry;  // [B, ng, S] scanned group totals or nullptr
    int64_t B, m;
    int g, suffix;
};

// In-place ordered binary-tree product of cnt signatures gs[0..cnt) (S floats each) held in
// shared memory by the whole CTA; the result ends in gs[0].  Level by level, top-down: a level-k
// update of the left operand reads only its levels < k and its own coefficient.
__device__ __forceinline__ void block_tree_combine(float* gs, int cnt, const TensorDims& d) {
    const int S = d.S;
    for (int stride = 1; stride < cnt; stride <<= 1) {
        const int npairs = (cnt + 2 * stride - 1) / (2 * stride);
        for (int k = d.N; k >= 1; --k) {
            const int nw = d.pw[k];
            for (int e = threadIdx.x; e < npairs * nw; e += blockDim.x) {
                const int pr = e / nw;
                const int w = e - pr * nw;
                const int left = pr * 2 * stride, right = left + stride;
                if (right >= cnt) continue;
                float* x = gs + left * S;
                const float* y = gs + right * S;
                x[d.off[k] + w] = mul_coef(d, x, y, k, w);
            }
            __syncthreads();
        }
    }
}

#ifdef SIG_DEFINE_COMBINE_KERNELS
__global__ void combine_group_kernel(const GroupParams p) {
    extern __shared__ float gs[];  // [G][S]
    const TensorDims& d = p.d;
    const int64_t g = blockIdx.x;
    const int64_t j0 = g * p.G;
    const int cnt = (int)((p.n - j0) < p.G ? (p.n - j0) : p.G);
    const int S = d.S;
    for (int64_t b = blockIdx.y; b < p.B; b += gridDim.y) {
        for (int jj = 0; jj < cnt; ++jj) {
            const float* src = p.in + (j0 + jj) * p.in_sj + b * p.in_sb;
            float* dst = gs + jj * S;
#pragma unroll 4
            for (int f = threadIdx.x; f < S; f += blockDim.x) dst[f] = __ldg(src + f);
        }
        __syncthreads();
        block_tree_combine(gs, cnt, d);
        float* o = p.out + g * p.out_sj + b * p.out_sb;
        for (int f = threadIdx.x; f < S; f += blockDim.x) o[f] = gs[f];
        __syncthreads();
    }
}

#endif  // SIG_DEFINE_COMBINE_KERNELS

}  // namespace sigb200

/*
 * oracle.c -- plain, slow, obviously-correct float64 CPU oracle for the Signatory hot path
 * (arXiv 2001.00706, "Signatory: differentiable computations of the signature and logsignature
 * transforms, on both CPU and GPU").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path (paper_2001_00706_b200/) never
 * links, imports or executes it, and this file shares no code, header, table or constant with
 * the CUDA path.
 *
 * Citations "P:Lnnn" are line numbers of /root/reference/PAPER.md (the paper's LaTeX source).
 *
 * Layout of a truncated tensor ("FreeTensor"): levels k = 1..N are stored
 * back to back (level-major); inside level k the word (j_1..j_k), 0-based letters, sits at
 * offset sum_m j_m * C^(k-m) (C-order flattening of the (C,)^k tensor).  The scalar level 0 is
 * implicit (P:L56 footnote): 1 for group elements (signatures), 0 for Lie elements (logs).
 *
 * Algorithms deliberately follow the plain definitions, not the paper's fused method:
 *  - exp(v) = (v, v^{(x)2}/2!, ..., v^{(x)N}/N!)
 *  - A [x] B level k = sum_{i=0}^{k} A_i (x) B_{k-i}, A_0 = B_0 = 1   P:L78-82 (eq-tensorproduct)
 *  - Sig(x_1..x_L) = exp(x_2-x_1) [x] ... [x] exp(x_L-x_{L-1})        P:L98-101 (eq-computation)
 *    evaluated as the "conventional way" of P:L333 (exp then [x], repeated), NOT Horner.
 *  - stream=True returns every prefix Sig(x_1..x_j), j = 2..L
 *  - the VJP is plain reverse-mode through that computation, storing every prefix; it does not use
 *    reversibility and so shares no algorithm with the CUDA backward.
 *  - log(1+x) = sum_{n=1}^{N} (-1)^{n+1} x^n / n, truncated, x^n by repeated products
 *    (P:L104-107 names log; the paper gives no algorithm, so the truncated series is the plain
 *    definition -- DESIGN.md reading R7).  Its VJP is plain reverse-mode through the series.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* C^k as int64 */
static int64_t ipow(int64_t C, int k) {
    int64_t r = 1;
    for (int i = 0; i < k; ++i) r *= C;
    return r;
}

/* S = sum_{k=1}^N C^k : the output width of the signature. */
int64_t orc_sig_channels(int C, int N) {
    int64_t s = 0;
    for (int k = 1; k <= N; ++k) s += ipow(C, k);
    return s;
}

/* offset of level k (1-based) in the flat layout */
int64_t orc_level_offset(int C, int k) {
    int64_t s = 0;
    for (int j = 1; j < k; ++j) s += ipow(C, j);
    return s;
}

/* ---------------------------------------------------------------------------------------------
 * exp: out level k = v^{(x)k} / k!.  Written out as the definition: the k-fold
 * outer product of v with itself, divided by k factorial.
 * ------------------------------------------------------------------------------------------- */
void orc_tensor_exp(const double* v, int C, int N, double* out) {
    double fact = 1.0;
    for (int k = 1; k <= N; ++k) {
        fact *= (double)k;
        double* lk = out + orc_level_offset(C, k);
        int64_t nk = ipow(C, k);
        for (int64_t w = 0; w < nk; ++w) {
            /* word w = (j_1..j_k): product of v[j_m] */
            double prod = 1.0;
            int64_t rem = w;
            for (int m = 0; m < k; ++m) {
                prod *= v[rem % C];
                rem /= C;
            }
            lk[w] = prod / fact;
        }
    }
}

/* ---------------------------------------------------------------------------------------------
 * Group-like product [x] (eq-tensorproduct P:L372-380):
 *   (A [x] B)_k = sum_{i=0}^{k} A_i (x) B_{k-i},  A_0 = a0, B_0 = b0 (scalars).
 * a0 = b0 = 1 for group elements.  a0 = b0 = 0 gives the plain product in the truncated tensor
 * algebra of two elements with zero scalar part (used by the log series).
 * Word (u v) with |u| = i, |v| = k-i has index u * C^{k-i} + v.
 * ------------------------------------------------------------------------------------------- */
void orc_mul_general(const double* a, double a0, const double* b, double b0, int C, int N,
                     double* out) {
    for (int k = 1; k <= N; ++k) {
        double* ok = out + orc_level_offset(C, k);
        int64_t nk = ipow(C, k);
        const double* ak = a + orc_level_offset(C, k);
        const double* bk = b + orc_level_offset(C, k);
        for (int64_t w = 0; w < nk; ++w) ok[w] = a0 * bk[w] + ak[w] * b0; /* i = 0 and i = k */
        for (int i = 1; i <= k - 1; ++i) {
            const double* ai = a + orc_level_offset(C, i);
            const double* bj = b + orc_level_offset(C, k - i);
            int64_t ni = ipow(C, i), nj = ipow(C, k - i);
            for (int64_t u = 0; u < ni; ++u)
                for (int64_t v = 0; v < nj; ++v) ok[u * nj + v] += ai[u] * bj[v];
        }
    }
}

void orc_mul(const double* a, const double* b, int C, int N, double* out) {
    orc_mul_general(a, 1.0, b, 1.0, C, N, out);
}

/* VJP of orc_mul_general w.r.t. a and b (scalars a0, b0 held fixed).  Accumulates (+=) into
 * ga and gb (either may be NULL).  Direct transposition of the double loop above. */
void orc_mul_general_vjp(const double* g, const double* a, double a0, const double* b, double b0,
                         int C, int N, double* ga, double* gb) {
    for (int k = 1; k <= N; ++k) {
        const double* gk = g + orc_level_offset(C, k);
        int64_t nk = ipow(C, k);
        if (ga) {
            double* gak = ga + orc_level_offset(C, k);
            for (int64_t w = 0; w < nk; ++w) gak[w] += gk[w] * b0;
        }
        if (gb) {
            double* gbk = gb + orc_level_offset(C, k);
            for (int64_t w = 0; w < nk; ++w) gbk[w] += a0 * gk[w];
        }
        for (int i = 1; i <= k - 1; ++i) {
            const double* ai = a + orc_level_offset(C, i);
            const double* bj = b + orc_level_offset(C, k - i);
            double* gai = ga ? ga + orc_level_offset(C, i) : NULL;
            double* gbj = gb ? gb + orc_level_offset(C, k - i) : NULL;
            int64_t ni = ipow(C, i), nj = ipow(C, k - i);
            for (int64_t u = 0; u < ni; ++u)
                for (int64_t v = 0; v < nj; ++v) {
                    double gw = gk[u * nj + v];
                    if (gai) gai[u] += gw * bj[v];
                    if (gbj) gbj[v] += ai[u] * gw;
                }
        }
    }
}

void orc_mul_vjp(const double* g, const double* a, const double* b, int C, int N, double* ga,
                 double* gb) {
    orc_mul_general_vjp(g, a, 1.0, b, 1.0, C, N, ga, gb);
}

/* VJP of orc_tensor_exp: plain reverse mode through E_k = E_{k-1} (x) v / k (E_0 = 1), which is
 * the definition v^{(x)k}/k! written as a recurrence.  Accumulates into gv[C]. */
void orc_tensor_exp_vjp(const double* g, const double* v, int C, int N, double* gv) {
    int64_t S = orc_sig_channels(C, N);
    double* E = (double*)malloc(sizeof(double) * (size_t)S);
    double* gE = (double*)malloc(sizeof(double) * (size_t)S);
    orc_tensor_exp(v, C, N, E);
    memcpy(gE, g, sizeof(double) * (size_t)S);
    for (int k = N; k >= 1; --k) {
        double* gk = gE + orc_level_offset(C, k);
        int64_t nprev = ipow(C, k - 1);
        if (k == 1) {
            for (int c = 0; c < C; ++c) gv[c] += gk[c]; /* E_1 = E_0 (x) v / 1 with E_0 = 1 */
        } else {
            const double* Ep = E + orc_level_offset(C, k - 1);
            double* gp = gE + orc_level_offset(C, k - 1);
            for (int64_t u = 0; u < nprev; ++u)
                for (int c = 0; c < C; ++c) {
                    double gw = gk[u * C + c] / (double)k;
                    gp[u] += gw * v[c];
                    gv[c] += Ep[u] * gw;
                }
        }
    }
    free(E);
    free(gE);
}

/* ---------------------------------------------------------------------------------------------
 * Signature of a stream (P:L68-75 dfn-stream-sig, P:L98-101 eq-computation), conventional way:
 *   P_1 = exp(z_0);  P_{t+1} = P_t [x] exp(z_t),   z_t = x_{t+1} - x_t,  t = 0..L-2.
 * path: [L, C] row-major.  stream = 0: out[S] = P_{L-1}.  stream = 1: out[L-1, S] = P_1..P_{L-1}
 * (the expanding intervals start at Sig(x_1, x_2)).
 * Any basepoint has already been prepended by the caller (reading R4).
 * Returns 0, or -1 if L < 2.
 * ------------------------------------------------------------------------------------------- */
int orc_signature(const double* path, int64_t L, int C, int N, int stream, double* out) {
    if (L < 2) return -1;
    int64_t S = orc_sig_channels(C, N);
    double* z = (double*)malloc(sizeof(double) * (size_t)C);
    double* E = (double*)malloc(sizeof(double) * (size_t)S);
    double* P = (double*)malloc(sizeof(double) * (size_t)S);
    double* Q = (double*)malloc(sizeof(double) * (size_t)S);
    for (int c = 0; c < C; ++c) z[c] = path[C + c] - path[c];
    orc_tensor_exp(z, C, N, P);
    if (stream) memcpy(out, P, sizeof(double) * (size_t)S);
    for (int64_t t = 1; t <= L - 2; ++t) {
        for (int c = 0; c < C; ++c) z[c] = path[(t + 1) * C + c] - path[t * C + c];
        orc_tensor_exp(z, C, N, E);
        orc_mul(P, E, C, N, Q);
        memcpy(P, Q, sizeof(double) * (size_t)S);
        if (stream) memcpy(out + t * S, P, sizeof(double) * (size_t)S);
    }
    if (!stream) memcpy(out, P, sizeof(double) * (size_t)S);
    free(z);
    free(E);
    free(P);
    free(Q);
    return 0;
}

/* ---------------------------------------------------------------------------------------------
 * VJP of orc_signature: plain reverse-mode through the conventional computation.  Stores every
 * prefix P_1..P_{L-1} and every exp(z_t) (O(L*S) memory), then walks back:
 *   (gP_t, gE_t) = VJP of [x] at (P_t, E_t);  gz_t = VJP of exp;  grad x_{t+1} += gz_t,
 *   grad x_t -= gz_t.
 * gout: [S] (stream = 0) or [L-1, S] (stream = 1: prefix j receives gout[j-1]).
 * gpath: [L, C], overwritten.
 * ------------------------------------------------------------------------------------------- */
int orc_signature_vjp(const double* gout, const double* path, int64_t L, int C, int N, int stream,
                      double* gpath) {
    if (L < 2) return -1;
    int64_t S = orc_sig_channels(C, N);
    int64_t M = L - 1;
    double* z = (double*)malloc(sizeof(double) * (size_t)(M * C));
    double* E = (double*)malloc(sizeof(double) * (size_t)(M * S)); /* E_t = exp(z_t) */
    double* P = (double*)malloc(sizeof(double) * (size_t)(M * S)); /* P_t = Sig(x_0..x_{t+1})*/
    double* G = (double*)malloc(sizeof(double) * (size_t)S);
    double* gP = (double*)malloc(sizeof(double) * (size_t)S);
    double* gE = (double*)malloc(sizeof(double) * (size_t)S);
    double* gz = (double*)malloc(sizeof(double) * (size_t)C);
    for (int64_t t = 0; t < M; ++t) {
        for (int c = 0; c < C; ++c) z[t * C + c] = path[(t + 1) * C + c] - path[t * C + c];
        orc_tensor_exp(z + t * C, C, N, E + t * S);
    }
    memcpy(P, E, sizeof(double) * (size_t)S);
    for (int64_t t = 1; t < M; ++t) orc_mul(P + (t - 1) * S, E + t * S, C, N, P + t * S);

    memset(gpath, 0, sizeof(double) * (size_t)(L * C));
    memset(G, 0, sizeof(double) * (size_t)S);
    for (int64_t t = M - 1; t >= 0; --t) {
        /* gradient arriving at P_t from the output */
        const double* go = stream ? gout + t * S : (t == M - 1 ? gout : NULL);
        if (go)
            for (int64_t s = 0; s < S; ++s) G[s] += go[s];
        memset(gE, 0, sizeof(double) * (size_t)S);
        if (t > 0) {
            memset(gP, 0, sizeof(double) * (size_t)S);
            orc_mul_vjp(G, P + (t - 1) * S, E + t * S, C, N, gP, gE);
        } else {
            memcpy(gE, G, sizeof(double) * (size_t)S); /* P_0 = E_0 */
        }
        memset(gz, 0, sizeof(double) * (size_t)C);
        orc_tensor_exp_vjp(gE, z + t * C, C, N, gz);
        for (int c = 0; c < C; ++c) {
            gpath[(t + 1) * C + c] += gz[c];
            gpath[t * C + c] -= gz[c];
        }
        if (t > 0) memcpy(G, gP, sizeof(double) * (size_t)S);
    }
    free(z);
    free(E);
    free(P);
    free(G);
    free(gP);
    free(gE);
    free(gz);
    return 0;
}

/* ---------------------------------------------------------------------------------------------
 * Tensor logarithm of a group element A (implicit scalar 1), P:L104-107 (eq-logarithm):
 *   x = A - 1 (scalar part 0);  log A = sum_{n=1}^{N} (-1)^{n+1} x^n / n   (truncated at N).
 * x^n by repeated products in the truncated algebra (orc_mul_general with zero scalars).
 * ------------------------------------------------------------------------------------------- */
void orc_log(const double* a, int C, int N, double* out) {
    int64_t S = orc_sig_channels(C, N);
    double* X = (double*)malloc(sizeof(double) * (size_t)S); /* x^n */
    double* Y = (double*)malloc(sizeof(double) * (size_t)S);
    memcpy(X, a, sizeof(double) * (size_t)S);
    memcpy(out, a, sizeof(double) * (size_t)S); /* n = 1 term */
    for (int n = 2; n <= N; ++n) {
        orc_mul_general(X, 0.0, a, 0.0, C, N, Y);
        memcpy(X, Y, sizeof(double) * (size_t)S);
        double coef = ((n % 2) ? 1.0 : -1.0) / (double)n;
        for (int64_t s = 0; s < S; ++s) out[s] += coef * X[s];
    }
    free(X);
    free(Y);
}

/* VJP of orc_log: reverse mode through the series above.  ga (size S) is overwritten. */
void orc_log_vjp(const double* g, const double* a, int C, int N, double* ga) {
    int64_t S = orc_sig_channels(C, N);
    /* forward: X_1 = a, X_n = X_{n-1} * a (stored) */
    double* X = (double*)malloc(sizeof(double) * (size_t)(S * (N + 1)));
    double* gX = (double*)malloc(sizeof(double) * (size_t)S);
    double* gXp = (double*)malloc(sizeof(double) * (size_t)S);
    memcpy(X + 1 * S, a, sizeof(double) * (size_t)S);
    for (int n = 2; n <= N; ++n) orc_mul_general(X + (n - 1) * S, 0.0, a, 0.0, C, N, X + n * S);
    memset(ga, 0, sizeof(double) * (size_t)S);
    /* gX_n = coef_n * g + (contribution from X_{n+1} = X_n * a) */
    memset(gX, 0, sizeof(double) * (size_t)S);
    for (int n = N; n >= 2; --n) {
        double coef = ((n % 2) ? 1.0 : -1.0) / (double)n;
        for (int64_t s = 0; s < S; ++s) gX[s] += coef * g[s];
        memset(gXp, 0, sizeof(double) * (size_t)S);
        orc_mul_general_vjp(gX, X + (n - 1) * S, 0.0, a, 0.0, C, N, gXp, ga);
        memcpy(gX, gXp, sizeof(double) * (size_t)S);
    }
    for (int64_t s = 0; s < S; ++s) ga[s] += gX[s] + g[s]; /* X_1 = a, coefficient 1 */
    free(X);
    free(gX);
    free(gXp);
}

/* Multiplication counts of Appendix A.1, exact integers; -1 on overflow.
 * conventional: C(d,N) = sum_{k=2}^N (d + binom(d+k-1, k)) + sum_{k=1}^N (k-1) d^k  (eq-conventional)
 * fused:        F(d,N) = d(N-1) + sum_{k=1}^N sum_{i=2}^k d^i                       (eq-fusedresult) */
int64_t orc_fused_cost(int64_t d, int N) {
    __int128 s = (__int128)d * (N - 1);
    for (int k = 1; k <= N; ++k)
        for (int i = 2; i <= k; ++i) {
            __int128 p = 1;
            for (int j = 0; j < i; ++j) p *= d;
            s += p;
        }
    if (s > (__int128)INT64_MAX) return -1;
    return (int64_t)s;
}

int64_t orc_conventional_cost(int64_t d, int N) {
    __int128 s = 0;
    for (int k = 2; k <= N; ++k) {
        /* binom(d+k-1, k) computed exactly by the multiplicative formula */
        __int128 b = 1;
        for (int j = 1; j <= k; ++j) b = b * (d + j - 1) / j;
        s += d + b;
    }
    for (int k = 1; k <= N; ++k) {
        __int128 p = 1;
        for (int j = 0; j < k; ++j) p *= d;
        s += (__int128)(k - 1) * p;
    }
    if (s > (__int128)INT64_MAX) return -1;
    return (int64_t)s;
}

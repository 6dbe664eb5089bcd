// lyndon.cpp -- host-side tables for the logsignature bases (Appendix A.2).
//
// * Lyndon words of length 1..N in (length, lex) order, generated with Duval's algorithm (each
//   word is produced once, in lex order, by the successor rule) -- not by filtering rotations.
// * Standard factorisation w = w^a w^b with w^b the longest proper Lyndon suffix.
// * phi(w) = [phi(w^a), phi(w^b)] as an integer combination of words.
// * M_k = psi o phi restricted to degree k is unit lower-triangular with integer entries
//   (P:L563-567); its inverse is therefore integer as well and is computed exactly (int64 forward
//   substitution), stored as CSR.  brackets = M^{-1} psi(log Sig) is then a sparse mat-vec on the
//   device instead of a sequential triangular solve.
#include "lyndon.h"

#include <algorithm>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <unordered_map>

namespace sigb200 {

namespace {

using Word = std::vector<int>;

int64_t word_index(const Word& w, int C) {
    int64_t idx = 0;
    for (int a : w) idx = idx * C + a;
    return idx;
}

// w is Lyndon iff it is strictly smaller than each of its proper suffixes (equivalent to the
// rotation definition of).
bool is_lyndon_word(const Word& w) {
    const int n = (int)w.size();
    for (int s = 1; s < n; ++s) {
        int a = 0, b = s;
        while (b < n && w[a] == w[b]) {
            ++a;
            ++b;
        }
        if (b == n) return false;      // the suffix is a prefix of w, hence smaller
        if (w[b] < w[a]) return false;  // the suffix is smaller
    }
    return true;
}

// Duval's generation: all Lyndon words of length <= N over {0..C-1} in lexicographic order.
std::vector<Word> duval_generate(int C, int N) {
    std::vector<Word> out;
    Word w{-1};
    while (!w.empty()) {
        w.back() += 1;
        out.push_back(w);
        const size_t m = w.size();
        while ((int)w.size() < N) w.push_back(w[w.size() - m]);
        while (!w.empty() && w.back() == C - 1) w.pop_back();
    }
    return out;
}

using Poly = std::map<Word, int64_t>;

Poly concat(const Poly& x, const Poly& y) {
    Poly r;
    for (auto& [u, a] : x)
        for (auto& [v, b] : y) {
            Word uv = u;
            uv.insert(uv.end(), v.begin(), v.end());
            r[uv] += a * b;
        }
    return r;
}

}  // namespace

LyndonTables build_lyndon_tables(int C, int N, bool need_brackets) {
    LyndonTables T;
    T.C = C;
    T.N = N;
    std::vector<Word> words = duval_generate(C, N);
    std::stable_sort(words.begin(), words.end(), [](const Word& a, const Word& b) {
        if (a.size() != b.size()) return a.size() < b.size();
        return a < b;
    });
    std::vector<int64_t> lvl_off(N + 2, 0);
    {
        int64_t p = 1;
        for (int k = 1; k <= N; ++k) {
            p *= C;
            lvl_off[k + 1] = lvl_off[k] + p;
        }
    }
    T.level_begin.assign(N + 2, 0);
    for (size_t j = 0; j < words.size(); ++j) {
        const int k = (int)words[j].size();
        T.flat_index.push_back(lvl_off[k] + word_index(words[j], C));
        T.level.push_back(k);
    }
    for (int k = 1; k <= N + 1; ++k) {
        T.level_begin[k] = (int)(std::lower_bound(T.level.begin(), T.level.end(), k) - T.level.begin());
    }
    T.level_begin[N + 1] = (int)words.size();
    if (!need_brackets) return T;

    // phi by recursion over the standard factorisation, memoised by word
    std::map<Word, Poly> memo;
    std::function<const Poly&(const Word&)> phi = [&](const Word& w) -> const Poly& {
        auto it = memo.find(w);
        if (it != memo.end()) return it->second;
        Poly p;
        if (w.size() == 1) {
            p[w] = 1;
        } else {
            size_t j = 1;
            for (; j < w.size(); ++j) {
                Word suf(w.begin() + j, w.end());
                if (is_lyndon_word(suf)) break;
            }
            Word a(w.begin(), w.begin() + j), b(w.begin() + j, w.end());
            const Poly pa = phi(a);
            const Poly pb = phi(b);
            Poly ab = concat(pa, pb), ba = concat(pb, pa);
            for (auto& [u, c] : ba) ab[u] -= c;
            for (auto& [u, c] : ab)
                if (c != 0) p[u] = c;
        }
        return memo.emplace(w, std::move(p)).first->second;
    };

    // per degree: M[r][c] = coefficient of Lyndon word r in phi(c), then exact integer inverse
    T.minv_rowptr.assign(1, 0);
    for (int k = 1; k <= N; ++k) {
        const int b0 = T.level_begin[k], b1 = T.level_begin[k + 1];
        const int n = b1 - b0;
        std::unordered_map<int64_t, int> pos;  // word index at level k -> row
        for (int r = 0; r < n; ++r) pos[word_index(words[b0 + r], C)] = r;
        // sparse columns of M: col c -> list (r, v)
        std::vector<std::vector<std::pair<int, int64_t>>> rows(n);  // rows[r] = (c, v), c <= r
        for (int c = 0; c < n; ++c) {
            for (auto& [u, v] : phi(words[b0 + c])) {
                auto it = pos.find(word_index(u, C));
                if (it != pos.end()) rows[it->second].push_back({c, v});
            }
        }
        for (int r = 0; r < n; ++r)
            for (auto& [c, v] : rows[r])
                if (c > r || (c == r && v != 1)) throw std::runtime_error("psi o phi is not unit lower-triangular");
        // X = M^{-1} by forward substitution, column by column: M x = e_j
        std::vector<std::vector<std::pair<int, int64_t>>> inv_rows(n);
        std::vector<int64_t> x(n);
        for (int j = 0; j < n; ++j) {
            std::fill(x.begin(), x.begin() + j, 0);
            for (int r = j; r < n; ++r) {
                int64_t acc = (r == j) ? 1 : 0;
                for (auto& [c, v] : rows[r])
                    if (c < r && c >= j) acc -= v * x[c];
                x[r] = acc;
                if (acc != 0) inv_rows[r].push_back({j, acc});
            }
        }
        for (int r = 0; r < n; ++r) {
            for (auto& [c, v] : inv_rows[r]) {
                T.minv_col.push_back(b0 + c);
                T.minv_val.push_back((double)v);
            }
            T.minv_rowptr.push_back((int)T.minv_col.size());
        }
        (void)b1;
    }
    // transpose (for the backward: g_psi = M^{-T} g_alpha)
    const int w = (int)words.size();
    std::vector<int> cnt(w + 1, 0);
    for (int c : T.minv_col) cnt[c + 1]++;
    for (int i = 0; i < w; ++i) cnt[i + 1] += cnt[i];
    T.minvT_rowptr = cnt;
    T.minvT_col.assign(T.minv_col.size(), 0);
    T.minvT_val.assign(T.minv_val.size(), 0.0);
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int r = 0; r < w; ++r)
        for (int e = T.minv_rowptr[r]; e < T.minv_rowptr[r + 1]; ++e) {
            const int c = T.minv_col[e];
            T.minvT_col[fill[c]] = r;
            T.minvT_val[fill[c]] = T.minv_val[e];
            fill[c]++;
        }
    return T;
}

int64_t witt_dimension(int64_t C, int N) {
    auto mobius = [](int n) {
        int r = 1, m = n;
        for (int p = 2; p * p <= m; ++p)
            if (m % p == 0) {
                m /= p;
                if (m % p == 0) return 0;
                r = -r;
            }
        return m > 1 ? -r : r;
    };
    __int128 tot = 0;
    for (int k = 1; k <= N; ++k) {
        __int128 s = 0;
        for (int i = 1; i <= k; ++i)
            if (k % i == 0) {
                __int128 p = 1;
                for (int j = 0; j < i; ++j) p *= C;
                s += mobius(k / i) * p;
            }
        tot += s / k;
    }
    if (tot > (__int128)INT64_MAX) return -1;
    return (int64_t)tot;
}

}  // namespace sigb200

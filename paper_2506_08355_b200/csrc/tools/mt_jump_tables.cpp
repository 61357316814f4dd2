// Build-time generator of the MT19937-64 jump-ahead polynomials used by rng.cu.
//
// The 312-word state window W_k = (x_k, ..., x_{k+311}) of mt19937_64 evolves linearly over
// GF(2): W_{k+1} = T W_k with x_{k+312} = x_{k+156} ^ twist(x_k, x_{k+1}).  On the 19937-bit
// part of the state that matters, T satisfies its characteristic polynomial p(x) (degree
// 19937, primitive), so T^J W = g_J(T) W with g_J = x^J mod p.  This program
//   1. recovers p by Berlekamp-Massey from one bit of the recurrence sequence,
//   2. tabulates g for J = a * 2^16 (a < 256, table A) and J = b * 2^24 (b < 256, table B),
//   3. checks every table entry class against plain sequential stepping,
// and writes them as a C++ source (coefficient i of g = bit i % 64 of word i / 64).
// Nothing here depends on the seed; the tables are constants of the generator.
#include <immintrin.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

namespace {

constexpr int kN = 312, kM = 156, kDeg = 19937, kWords = 312;  // 312 * 64 = 19968 >= 19937
constexpr uint64_t kUm = 0xFFFFFFFF80000000ULL, kLm = 0x7FFFFFFFULL, kA = 0xB5026F5AA96619E9ULL;
constexpr int kLogJ0 = 16;  // table A stride: 65536 draws

using Poly = std::vector<uint64_t>;

inline uint64_t twist(uint64_t a, uint64_t b) {
    const uint64_t x = (a & kUm) | (b & kLm);
    return (x >> 1) ^ ((0ULL - (x & 1ULL)) & kA);
}

// y[0..311] = window; extend the sequence to `len` words.
void extend(std::vector<uint64_t>& y, size_t len) {
    y.resize(len);
    for (size_t m = kN; m < len; ++m) y[m] = y[m - kN + kM] ^ twist(y[m - kN], y[m - kN + 1]);
}

inline int bit(const Poly& p, int i) { return static_cast<int>((p[i >> 6] >> (i & 63)) & 1ULL); }
inline void flip(Poly& p, int i) { p[i >> 6] ^= 1ULL << (i & 63); }

int degree(const Poly& p) {
    for (int w = static_cast<int>(p.size()) - 1; w >= 0; --w)
        if (p[w]) return w * 64 + 63 - __builtin_clzll(p[w]);
    return -1;
}

// Berlekamp-Massey over GF(2): connection polynomial C (C_0 = 1) of the bit sequence s.
Poly berlekamp_massey(const std::vector<uint8_t>& s, int& len) {
    const int n = static_cast<int>(s.size());
    const int words = (n + 64) / 64 + 1;
    Poly c(words, 0), b(words, 0), t;
    c[0] = b[0] = 1;
    int l = 0, m = 1;
    for (int k = 0; k < n; ++k) {
        int d = s[k];
        for (int i = 1; i <= l; ++i) d ^= bit(c, i) & s[k - i];
        if (!d) {
            ++m;
            continue;
        }
        t = c;
        // c += x^m b
        const int ws = m >> 6, bs = m & 63;
        for (int w = words - 1; w >= ws; --w) {
            uint64_t v = b[w - ws] << bs;
            if (bs && w - ws - 1 >= 0) v |= b[w - ws - 1] >> (64 - bs);
            c[w] ^= v;
        }
        if (2 * l <= k) {
            l = k + 1 - l;
            b = t;
            m = 1;
        } else {
            ++m;
        }
    }
    len = l;
    return c;
}

struct Field {
    Poly p;                         // characteristic polynomial, degree kDeg
    std::vector<Poly> shifted;      // p << s for s = 0..63, kWords + 1 words each

    void init(const Poly& pp) {
        p = pp;
        p.resize(kWords + 1, 0);
        shifted.assign(64, Poly(kWords + 2, 0));
        for (int s = 0; s < 64; ++s)
            for (int w = 0; w <= kWords; ++w) {
                shifted[s][w] ^= p[w] << s;
                if (s) shifted[s][w + 1] ^= p[w] >> (64 - s);
            }
    }
    // r (2 * kWords words, degree < 2 * kDeg) mod p -> kWords words
    Poly reduce(Poly r) const {
        for (int i = 2 * kWords * 64 - 1; i >= kDeg; --i) {
            if (!((r[i >> 6] >> (i & 63)) & 1ULL)) continue;
            const int sh = i - kDeg, ws = sh >> 6, bs = sh & 63;
            const Poly& q = shifted[bs];
            for (int w = 0; w < kWords + 2 && ws + w < static_cast<int>(r.size()); ++w) r[ws + w] ^= q[w];
        }
        r.resize(kWords);
        return r;
    }
    Poly mul(const Poly& a, const Poly& b) const {
        Poly r(2 * kWords + 2, 0);
        for (int i = 0; i < kWords; ++i) {
            if (!a[i]) continue;
            const __m128i ai = _mm_set_epi64x(0, static_cast<long long>(a[i]));
            for (int j = 0; j < kWords; ++j) {
                if (!b[j]) continue;
                const __m128i bj = _mm_set_epi64x(0, static_cast<long long>(b[j]));
                const __m128i pr = _mm_clmulepi64_si128(ai, bj, 0);
                r[i + j] ^= static_cast<uint64_t>(_mm_cvtsi128_si64(pr));
                r[i + j + 1] ^= static_cast<uint64_t>(_mm_extract_epi64(pr, 1));
            }
        }
        return reduce(r);
    }
};

// g(T) W by correlation: word j of the result = XOR over set coefficients i of y_{i+j}.
std::vector<uint64_t> jump(const Poly& g, const std::vector<uint64_t>& w) {
    std::vector<uint64_t> y(w.begin(), w.end());
    extend(y, kDeg + kN + 1);
    std::vector<uint64_t> out(kN, 0);
    for (int i = 0; i < kDeg; ++i)
        if (bit(g, i))
            for (int j = 0; j < kN; ++j) out[j] ^= y[i + j];
    return out;
}

// Window after `count` single steps, computed by extending the sequence.
std::vector<uint64_t> advance_window(const std::vector<uint64_t>& w, uint64_t count) {
    std::vector<uint64_t> y(w);
    extend(y, count + kN);
    return std::vector<uint64_t>(y.begin() + count, y.begin() + count + kN);
}

bool same_future(const std::vector<uint64_t>& a, const std::vector<uint64_t>& b) {
    // windows are equivalent when they agree on every bit that influences later outputs:
    // all of x_{k+1..k+311} and the upper 33 bits of x_k
    if ((a[0] & kUm) != (b[0] & kUm)) return false;
    for (int i = 1; i < kN; ++i)
        if (a[i] != b[i]) return false;
    return true;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc != 2) {
        std::fprintf(stderr, "usage: %s out.cpp\n", argv[0]);
        return 2;
    }
    // 1. characteristic polynomial from bit 0 of the recurrence sequence
    std::vector<uint64_t> w0(kN);
    {
        std::mt19937_64 eng(5489ULL);
        for (int i = 0; i < kN; ++i) w0[i] = eng();
    }
    std::vector<uint64_t> y(w0);
    const int nbits = 2 * kDeg + 200;
    extend(y, nbits + kN);
    std::vector<uint8_t> s(nbits);
    for (int k = 0; k < nbits; ++k) s[k] = static_cast<uint8_t>(y[k + kN] & 1ULL);
    int l = 0;
    Poly c = berlekamp_massey(s, l);
    if (l != kDeg) {
        std::fprintf(stderr, "mt_jump_tables: linear complexity %d, expected %d\n", l, kDeg);
        return 1;
    }
    Poly p(kWords + 1, 0);
    for (int j = 0; j <= kDeg; ++j)
        if (bit(c, kDeg - j)) flip(p, j);
    Field f;
    f.init(p);

    // 2. x^(2^16) by squaring, table A = x^(a 2^16), table B = x^(b 2^24)
    Poly x(kWords, 0);
    x[0] = 2ULL;
    Poly g0 = x;
    for (int i = 0; i < kLogJ0; ++i) g0 = f.mul(g0, g0);
    std::vector<Poly> ta(256), tb(256);
    ta[0] = Poly(kWords, 0);
    ta[0][0] = 1ULL;
    for (int a = 1; a < 256; ++a) ta[a] = f.mul(ta[a - 1], g0);
    const Poly g1 = f.mul(ta[255], g0);  // x^(256 * 2^16)
    tb[0] = ta[0];
    for (int b = 1; b < 256; ++b) tb[b] = f.mul(tb[b - 1], g1);

    // 3. checks against sequential stepping
    std::mt19937_64 chk(12345ULL);
    std::vector<uint64_t> w(kN);
    for (auto& v : w) v = chk();
    for (int a : {1, 2, 7, 255}) {
        if (!same_future(jump(ta[a], w), advance_window(w, static_cast<uint64_t>(a) << kLogJ0))) {
            std::fprintf(stderr, "mt_jump_tables: table A[%d] check failed\n", a);
            return 1;
        }
    }
    {
        const std::vector<uint64_t> j1 = jump(tb[1], w);
        if (!same_future(j1, advance_window(w, 1ULL << 24))) {
            std::fprintf(stderr, "mt_jump_tables: table B[1] check failed\n");
            return 1;
        }
        const std::vector<uint64_t> j3 = jump(ta[3], jump(tb[2], w));
        if (!same_future(j3, advance_window(w, (2ULL << 24) + (3ULL << 16)))) {
            std::fprintf(stderr, "mt_jump_tables: table B[2]A[3] check failed\n");
            return 1;
        }
    }
    
    FILE* o = std::fopen(argv[1], "w");
    if (!o) return 1;
    std::fprintf(o, "// Generated by tools/mt_jump_tables.cpp -- MT19937-64 jump polynomials.\n");
    std::fprintf(o, "#include <cstdint>\nnamespace bosp {\ninline namespace b200 {\n");
    std::fprintf(o, "extern const uint64_t kMtJump[2][256][%d];\n", kWords);
    std::fprintf(o, "const uint64_t kMtJump[2][256][%d] = {\n", kWords);
    for (int t = 0; t < 2; ++t) {
        std::fprintf(o, "{\n");
        for (int a = 0; a < 256; ++a) {
            const Poly& g = t == 0 ? ta[a] : tb[a];
            std::fprintf(o, "{");
            for (int i = 0; i < kWords; ++i) std::fprintf(o, "0x%llxULL,", static_cast<unsigned long long>(g[i]));
            std::fprintf(o, "},\n");
        }
        std::fprintf(o, "},\n");
    }
    std::fprintf(o, "};\n}  // namespace b200\n}  // namespace bosp\n");
    std::fclose(o);
    return 0;
}

// host_mt.h -- jump-ahead for the mt19937_64 stream of the generators.
//
// gen_congested (gen.hpp:103-128) draws one Bernoulli per (hot link, stream)
// pair from ONE sequential mt19937_64 stream: at config C scale that is
// 1e10 draws, ~30 s on one core.  The draw for pair (i, j) is raw output
// number P0 + i*n + j, so any contiguous range of pairs can be drawn on its
// own thread once the engine state at its first position is known.  That
// state comes from a jump: the engine is linear over GF(2), its transition
// A has characteristic polynomial phi (degree 19937), and the state J
// outputs ahead is p(A) w with p(x) = x^J mod phi(x) (Horner over p's
// coefficients, one engine step each).  phi is recovered once per process
// by Berlekamp-Massey from 2 * 19937 output bits.  Every draw is the one
// the sequential engine would have made: tests/test_host.py checks the
// jumped engine against std::mt19937_64 and the generator against the
// reference's.
//
// Engine constants and seeding are those the C++ standard pins for
// mt19937_64 ([rand.predef]); the window representation below is the
// standard's textual state: the last n = 312 raw words produced.
#pragma once

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

namespace numpmp_mt {

constexpr int kN = 312, kM = 156, kDeg = 19937;
constexpr std::uint64_t kA = 0xB5026F5AA96619E9ULL;
constexpr std::uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;

inline std::uint64_t temper(std::uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

inline std::uint64_t mix(std::uint64_t xk, std::uint64_t xk1, std::uint64_t xkm) {
  const std::uint64_t y = (xk & kUpper) | (xk1 & kLower);
  return xkm ^ (y >> 1) ^ ((y & 1) ? kA : 0);
}

// The window of the seeded engine (position 0: no output drawn yet).
inline void seed_window(std::uint64_t seed, std::uint64_t* w) {
  w[0] = seed;
  for (int i = 1; i < kN; ++i)
    w[i] = 6364136223846793005ULL * (w[i - 1] ^ (w[i - 1] >> 62)) + static_cast<std::uint64_t>(i);
}

// Block engine started from a window: draws the outputs that follow it.
class Engine {
 public:
  explicit Engine(const std::uint64_t* window) {
    std::memcpy(mt_, window, sizeof(mt_));
    idx_ = kN;
  }
  std::uint64_t operator()() {
    if (idx_ >= kN) twist();
    return temper(mt_[idx_++]);
  }

 private:
  void twist() {
    for (int i = 0; i < kN - kM; ++i) mt_[i] = mix(mt_[i], mt_[i + 1], mt_[i + kM]);
    for (int i = kN - kM; i < kN - 1; ++i) mt_[i] = mix(mt_[i], mt_[i + 1], mt_[i + kM - kN]);
    mt_[kN - 1] = mix(mt_[kN - 1], mt_[0], mt_[kM - 1]);
    idx_ = 0;
  }
  std::uint64_t mt_[kN];
  int idx_;
};

namespace detail {

constexpr int kW = (2 * kDeg + 63) / 64 + 1;  // words of a product before reduction
constexpr int kPW = (kDeg + 1 + 63) / 64;     // words of a reduced polynomial (deg <= kDeg)

using Poly = std::vector<std::uint64_t>;

inline bool bit(const Poly& p, long i) { return (p[static_cast<std::size_t>(i >> 6)] >> (i & 63)) & 1; }

// phi from Berlekamp-Massey over bit 0 of successive raw words (a linear
// functional of the state, so the sequence satisfies phi(A)).  Returns the
// monic characteristic polynomial x^L + c_1 x^(L-1) + ... + c_L.
inline Poly char_poly() {
  const int N = 2 * kDeg + 64;
  std::vector<std::uint8_t> s(static_cast<std::size_t>(N));
  {
    std::uint64_t w[kN];
    seed_window(5489u, w);
    // incremental steps: s_k = bit 0 of raw word x_{n+k}
    int h = 0;
    for (int k = 0; k < N; ++k) {
      const std::uint64_t x = mix(w[h], w[(h + 1) % kN], w[(h + kM) % kN]);
      w[h] = x;
      h = (h + 1) % kN;
      s[static_cast<std::size_t>(k)] = static_cast<std::uint8_t>(x & 1);
    }
  }
  const int W = (N + 63) / 64 + 1;
  Poly C(W, 0), B(W, 0), T(W, 0), R(W, 0);  // R bit i = s_{n-i}
  C[0] = B[0] = 1;
  int L = 0, m = 1;
  auto shl1_in = [&](Poly& r, std::uint64_t in) {
    for (int i = W - 1; i > 0; --i) r[i] = (r[i] << 1) | (r[i - 1] >> 63);
    r[0] = (r[0] << 1) | in;
  };
  auto xor_shifted = [&](Poly& dst, const Poly& src, int sh) {
    const int ws = sh >> 6, bs = sh & 63;
    for (int i = W - 1; i >= ws; --i) {
      std::uint64_t v = src[i - ws] << bs;
      if (bs && i - ws - 1 >= 0) v |= src[i - ws - 1] >> (64 - bs);
      dst[i] ^= v;
    }
  };
  for (int n = 0; n < N; ++n) {
    shl1_in(R, s[static_cast<std::size_t>(n)]);
    const int lw = L / 64 + 1;
    std::uint64_t acc = 0;
    for (int i = 0; i < lw && i < W; ++i) acc ^= C[i] & R[i];
    const int d = __builtin_parityll(acc);
    if (d == 0) {
      ++m;
    } else if (2 * L <= n) {
      T = C;
      xor_shifted(C, B, m);
      L = n + 1 - L;
      B = T;
      m = 1;
    } else {
      xor_shifted(C, B, m);
      ++m;
    }
  }
  Poly phi(kPW, 0);  // reverse of C(x) = 1 + c_1 x + ... + c_L x^L
  for (int i = 0; i <= L; ++i)
    if (bit(C, i)) phi[static_cast<std::size_t>((L - i) >> 6)] |= 1ULL << ((L - i) & 63);
  if (L != kDeg) phi.clear();  // cannot happen for mt19937_64; caller checks
  return phi;
}

inline const Poly& phi() {
  static Poly p;
  static std::once_flag once;
  std::call_once(once, [] { p = char_poly(); });
  return p;
}

// r = r mod phi for r of kW words (degree < 2 * kDeg).
inline void reduce(Poly& r, const std::vector<Poly>& phi_sh) {
  for (long d = static_cast<long>(kW) * 64 - 1; d >= kDeg; --d) {
    if (!bit(r, d)) continue;
    const long sh = d - kDeg;  // r ^= phi << sh
    const Poly& ps = phi_sh[static_cast<std::size_t>(sh & 63)];
    const long ws = sh >> 6;
    for (long i = 0; i < static_cast<long>(ps.size()) && i + ws < kW; ++i)
      r[static_cast<std::size_t>(i + ws)] ^= ps[static_cast<std::size_t>(i)];
  }
}

// x^J mod phi
inline Poly x_pow_mod(std::uint64_t J) {
  const Poly& ph = phi();
  std::vector<Poly> phi_sh(64);
  for (int s = 0; s < 64; ++s) {
    Poly q(kPW + 1, 0);
    for (int i = 0; i < kPW; ++i) {
      q[static_cast<std::size_t>(i)] |= ph[static_cast<std::size_t>(i)] << s;
      if (s) q[static_cast<std::size_t>(i) + 1] |= ph[static_cast<std::size_t>(i)] >> (64 - s);
    }
    phi_sh[static_cast<std::size_t>(s)] = q;
  }
  Poly r(kW, 0);
  r[0] = 1;
  for (int b = 63; b >= 0; --b) {
    if (r[0] != 1 || std::count(r.begin(), r.end(), 0ULL) != kW - 1) {  // r != 1: square
      Poly sq(kW, 0);  // spread the bits of r into the even positions
      for (int i = 0; i < kPW; ++i) {
        const std::uint64_t v = r[static_cast<std::size_t>(i)];
        std::uint64_t lo = 0, hi = 0;
        for (int k = 0; k < 32; ++k) {
          lo |= ((v >> k) & 1ULL) << (2 * k);
          hi |= ((v >> (k + 32)) & 1ULL) << (2 * k);
        }
        sq[static_cast<std::size_t>(2 * i)] ^= lo;
        if (2 * i + 1 < kW) sq[static_cast<std::size_t>(2 * i + 1)] ^= hi;
      }
      reduce(sq, phi_sh);
      r.swap(sq);
    }
    if ((J >> b) & 1) {  // * x
      for (int i = kW - 1; i > 0; --i) r[i] = (r[i] << 1) | (r[i - 1] >> 63);
      r[0] <<= 1;
      reduce(r, phi_sh);
    }
  }
  r.resize(kPW);
  return r;
}

}  // namespace detail

// The window J outputs after `window` (J >= 0).  Returns false if phi could
// not be recovered (never for mt19937_64).
inline bool jump(const std::uint64_t* window, std::uint64_t J, std::uint64_t* out) {
  if (J == 0) {
    std::memcpy(out, window, sizeof(std::uint64_t) * kN);
    return true;
  }
  if (detail::phi().empty()) return false;
  const detail::Poly p = detail::x_pow_mod(J);
  // Horner: acc = A acc + p_i w, i = deg .. 0, on a circular window
  std::uint64_t acc[kN] = {};
  int h = 0;  // acc's oldest word
  for (int i = kDeg - 1; i >= 0; --i) {
    acc[h] = mix(acc[h], acc[(h + 1) % kN], acc[(h + kM) % kN]);
    h = (h + 1) % kN;
    if (detail::bit(p, i))
      for (int t = 0, q = h; t < kN; ++t, q = (q + 1 == kN ? 0 : q + 1)) acc[q] ^= window[t];
  }
  for (int t = 0; t < kN; ++t) out[t] = acc[(h + t) % kN];
  return true;
}

}  // namespace numpmp_mt

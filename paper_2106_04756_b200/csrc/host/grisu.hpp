// grisu.hpp -- decimal digits of a double as the reference's JSON writer
// prints them.
//
// The reference serializes results through nlohmann::json (result_io.cpp:53-98),
// whose number output is Loitsch's Grisu2 ("Printing Floating-Point Numbers
// Quickly and Accurately with Integers", PLDI 2010) with the alpha/gamma =
// -60/-32 window and 8-decade cached powers.  Grisu2 always round-trips but
// is not always the SHORTEST representation (e.g. 0.0012036080000000001 where
// the shortest is 0.001203608), so std::to_chars cannot reproduce the
// reference's bytes.  This is a restatement of the published algorithm:
//   1. v = f * 2^e and the midpoints m-, m+ to its neighbours, all scaled to
//      one binary exponent;
//   2. a cached power c ~ 10^-k that brings that exponent into [-60, -32];
//   3. the products w = v*c, M- = m-*c + 1 ulp, M+ = m+*c - 1 ulp (64x64-bit
//      multiplies, rounded), i.e. a safe interval around v*10^-k;
//   4. digits of M+ until the remainder drops inside the interval, then the
//      last digit is walked down toward w while that stays inside and gets
//      closer ("weeding").
// The cached-power table below was generated with exact rational arithmetic
// (10^k, k = -300, -292, ..., 324, significand rounded to nearest 64 bits).
// tests/test_mps.py checks the writer byte for byte against the reference on
// random and adversarial doubles.
#pragma once

#include <cstdint>
#include <cstring>

namespace folp::grisu {

struct Fp {
  uint64_t f;
  int e;
};

inline Fp mul(Fp x, Fp y) {
  const unsigned __int128 p = static_cast<unsigned __int128>(x.f) * y.f;
  uint64_t hi = static_cast<uint64_t>(p >> 64);
  const uint64_t lo = static_cast<uint64_t>(p);
  hi += lo >> 63;  // round half up
  return Fp{hi, x.e + y.e + 64};
}

inline Fp normalize(Fp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}

struct CachedPower {
  uint64_t f;
  int e;
  int k;
};

inline const CachedPower& cached_power(int e) {
  static const CachedPower table[] = {
    {0xAB70FE17C79AC6CAull, -1060, -300},
    {0xFF77B1FCBEBCDC4Full, -1034, -292},
    {0xBE5691EF416BD60Cull, -1007, -284},
    {0x8DD01FAD907FFC3Cull, -980, -276},
    {0xD3515C2831559A83ull, -954, -268},
    {0x9D71AC8FADA6C9B5ull, -927, -260},
    {0xEA9C227723EE8BCBull, -901, -252},
    {0xAECC49914078536Dull, -874, -244},
    {0x823C12795DB6CE57ull, -847, -236},
    {0xC21094364DFB5637ull, -821, -228},
    {0x9096EA6F3848984Full, -794, -220},
    {0xD77485CB25823AC7ull, -768, -212},
    {0xA086CFCD97BF97F4ull, -741, -204},
    {0xEF340A98172AACE5ull, -715, -196},
    {0xB23867FB2A35B28Eull, -688, -188},
    {0x84C8D4DFD2C63F3Bull, -661, -180},
    {0xC5DD44271AD3CDBAull, -635, -172},
    {0x936B9FCEBB25C996ull, -608, -164},
    {0xDBAC6C247D62A584ull, -582, -156},
    {0xA3AB66580D5FDAF6ull, -555, -148},
    {0xF3E2F893DEC3F126ull, -529, -140},
    {0xB5B5ADA8AAFF80B8ull, -502, -132},
    {0x87625F056C7C4A8Bull, -475, -124},
    {0xC9BCFF6034C13053ull, -449, -116},
    {0x964E858C91BA2655ull, -422, -108},
    {0xDFF9772470297EBDull, -396, -100},
    {0xA6DFBD9FB8E5B88Full, -369, -92},
    {0xF8A95FCF88747D94ull, -343, -84},
    {0xB94470938FA89BCFull, -316, -76},
    {0x8A08F0F8BF0F156Bull, -289, -68},
    {0xCDB02555653131B6ull, -263, -60},
    {0x993FE2C6D07B7FACull, -236, -52},
    {0xE45C10C42A2B3B06ull, -210, -44},
    {0xAA242499697392D3ull, -183, -36},
    {0xFD87B5F28300CA0Eull, -157, -28},
    {0xBCE5086492111AEBull, -130, -20},
    {0x8CBCCC096F5088CCull, -103, -12},
    {0xD1B71758E219652Cull, -77, -4},
    {0x9C40000000000000ull, -50, 4},
    {0xE8D4A51000000000ull, -24, 12},
    {0xAD78EBC5AC620000ull, 3, 20},
    {0x813F3978F8940984ull, 30, 28},
    {0xC097CE7BC90715B3ull, 56, 36},
    {0x8F7E32CE7BEA5C70ull, 83, 44},
    {0xD5D238A4ABE98068ull, 109, 52},
    {0x9F4F2726179A2245ull, 136, 60},
    {0xED63A231D4C4FB27ull, 162, 68},
    {0xB0DE65388CC8ADA8ull, 189, 76},
    {0x83C7088E1AAB65DBull, 216, 84},
    {0xC45D1DF942711D9Aull, 242, 92},
    {0x924D692CA61BE758ull, 269, 100},
    {0xDA01EE641A708DEAull, 295, 108},
    {0xA26DA3999AEF774Aull, 322, 116},
    {0xF209787BB47D6B85ull, 348, 124},
    {0xB454E4A179DD1877ull, 375, 132},
    {0x865B86925B9BC5C2ull, 402, 140},
    {0xC83553C5C8965D3Dull, 428, 148},
    {0x952AB45CFA97A0B3ull, 455, 156},
    {0xDE469FBD99A05FE3ull, 481, 164},
    {0xA59BC234DB398C25ull, 508, 172},
    {0xF6C69A72A3989F5Cull, 534, 180},
    {0xB7DCBF5354E9BECEull, 561, 188},
    {0x88FCF317F22241E2ull, 588, 196},
    {0xCC20CE9BD35C78A5ull, 614, 204},
    {0x98165AF37B2153DFull, 641, 212},
    {0xE2A0B5DC971F303Aull, 667, 220},
    {0xA8D9D1535CE3B396ull, 694, 228},
    {0xFB9B7CD9A4A7443Cull, 720, 236},
    {0xBB764C4CA7A44410ull, 747, 244},
    {0x8BAB8EEFB6409C1Aull, 774, 252},
    {0xD01FEF10A657842Cull, 800, 260},
    {0x9B10A4E5E9913129ull, 827, 268},
    {0xE7109BFBA19C0C9Dull, 853, 276},
    {0xAC2820D9623BF429ull, 880, 284},
    {0x80444B5E7AA7CF85ull, 907, 292},
    {0xBF21E44003ACDD2Dull, 933, 300},
    {0x8E679C2F5E44FF8Full, 960, 308},
    {0xD433179D9C8CB841ull, 986, 316},
    {0x9E19DB92B4E31BA9ull, 1013, 324}
  };
  // the smallest 10^k with alpha <= e + e_c + 64 (alpha = -60):
  // k = ceil((alpha - e - 1) * log10(2))
  const int f = -60 - e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);
  const int index = (300 + k + 7) / 8;
  return table[index];
}

inline void weed(char* buf, int len, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
  while (rest < dist && delta - rest >= ten_k &&
         (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    --buf[len - 1];
    rest += ten_k;
  }
}

// Digits of v (finite, > 0) into buf (>= 18 chars); value = digits * 10^K.
// Returns the digit count.
inline int digits(double v, char* buf, int& K) {
  uint64_t bits;
  std::memcpy(&bits, &v, sizeof bits);
  const uint64_t F = bits & ((uint64_t{1} << 52) - 1);
  const int E = static_cast<int>(bits >> 52) & 0x7ff;
  const Fp x = E == 0 ? Fp{F, -1074} : Fp{F + (uint64_t{1} << 52), E - 1075};
  const bool closer = F == 0 && E > 1;  // the lower neighbour is half as far
  const Fp mp = normalize(Fp{2 * x.f + 1, x.e - 1});
  Fp mm = closer ? Fp{4 * x.f - 1, x.e - 2} : Fp{2 * x.f - 1, x.e - 1};
  mm.f <<= (mm.e - mp.e);
  mm.e = mp.e;
  const Fp w = normalize(x);
  const CachedPower& c = cached_power(mp.e);
  const Fp cp{c.f, c.e};
  const Fp W = mul(w, cp);
  Fp lo = mul(mm, cp), hi = mul(mp, cp);
  ++lo.f;
  --hi.f;
  K = -c.k;
  uint64_t delta = hi.f - lo.f;
  uint64_t dist = hi.f - W.f;
  const int sh = -hi.e;
  const uint64_t one = uint64_t{1} << sh;
  uint32_t p1 = static_cast<uint32_t>(hi.f >> sh);
  uint64_t p2 = hi.f & (one - 1);
  int n = 1;
  uint32_t pow10 = 1;
  while (n < 10 && p1 >= pow10 * 10u) {
    pow10 *= 10u;
    ++n;
  }
  int len = 0;
  while (n > 0) {
    const uint32_t d = p1 / pow10;
    p1 %= pow10;
    buf[len++] = static_cast<char>('0' + d);
    --n;
    const uint64_t rest = (static_cast<uint64_t>(p1) << sh) + p2;
    if (rest <= delta) {
      K += n;
      weed(buf, len, dist, delta, rest, static_cast<uint64_t>(pow10) << sh);
      return len;
    }
    pow10 /= 10u;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    const uint64_t d = p2 >> sh;
    p2 &= one - 1;
    buf[len++] = static_cast<char>('0' + d);
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  K -= m;
  weed(buf, len, dist, delta, p2, one);
  return len;
}

}  // namespace folp::grisu

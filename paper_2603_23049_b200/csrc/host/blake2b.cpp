// BLAKE2b as specified by RFC 7693 §3 (compression F, §3.2) with the parameter block of
// §2.5 reduced to digest length and key length (no salt/personalisation).
#include "blake2b.h"

#include <cstring>

namespace pcr {
namespace {

constexpr uint64_t kIV[8] = {
    0x6A09E667F3BCC908ULL, 0xBB67AE8584CAA73BULL, 0x3C6EF372FE94F82BULL, 0xA54FF53A5F1D36F1ULL,
    0x510E527FADE682D1ULL, 0x9B05688C2B3E6C1FULL, 0x1F83D9ABFB41BD6BULL, 0x5BE0CD19137E2179ULL};

constexpr uint8_t kSigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4},
    {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13},
    {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11},
    {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5},
    {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15},
    {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

inline uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

inline uint64_t load64le(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

// RFC 7693 §3.1 mixing function G.
inline void G(uint64_t* v, int a, int b, int c, int d, uint64_t x, uint64_t y) {
  v[a] = v[a] + v[b] + x;
  v[d] = rotr64(v[d] ^ v[a], 32);
  v[c] = v[c] + v[d];
  v[b] = rotr64(v[b] ^ v[c], 24);
  v[a] = v[a] + v[b] + y;
  v[d] = rotr64(v[d] ^ v[a], 16);
  v[c] = v[c] + v[d];
  v[b] = rotr64(v[b] ^ v[c], 63);
}

// RFC 7693 §3.2 compression function F.
void compress(Blake2b* s, bool last) {
  uint64_t v[16], m[16];
  for (int i = 0; i < 8; ++i) {
    v[i] = s->h[i];
    v[i + 8] = kIV[i];
  }
  v[12] ^= s->t[0];
  v[13] ^= s->t[1];
  if (last) v[14] = ~v[14];
  for (int i = 0; i < 16; ++i) m[i] = load64le(s->buf + 8 * i);
  for (int r = 0; r < 12; ++r) {
    const uint8_t* sg = kSigma[r];
    G(v, 0, 4, 8, 12, m[sg[0]], m[sg[1]]);
    G(v, 1, 5, 9, 13, m[sg[2]], m[sg[3]]);
    G(v, 2, 6, 10, 14, m[sg[4]], m[sg[5]]);
    G(v, 3, 7, 11, 15, m[sg[6]], m[sg[7]]);
    G(v, 0, 5, 10, 15, m[sg[8]], m[sg[9]]);
    G(v, 1, 6, 11, 12, m[sg[10]], m[sg[11]]);
    G(v, 2, 7, 8, 13, m[sg[12]], m[sg[13]]);
    G(v, 3, 4, 9, 14, m[sg[14]], m[sg[15]]);
  }
  for (int i = 0; i < 8; ++i) s->h[i] ^= v[i] ^ v[i + 8];
}

}  // namespace

bool blake2b_init(Blake2b* s, size_t outlen, const void* key, size_t keylen) {
  if (outlen == 0 || outlen > 64 || keylen > 64) return false;
  for (int i = 0; i < 8; ++i) s->h[i] = kIV[i];
  s->h[0] ^= 0x01010000ULL ^ (static_cast<uint64_t>(keylen) << 8) ^ outlen;
  s->t[0] = s->t[1] = 0;
  s->c = 0;
  s->outlen = outlen;
  std::memset(s->buf, 0, sizeof(s->buf));
  if (keylen > 0) {
    blake2b_update(s, key, keylen);
    s->c = 128;  // a full key block, padded with zeros
  }
  return true;
}

void blake2b_update(Blake2b* s, const void* in, size_t inlen) {
  const uint8_t* p = static_cast<const uint8_t*>(in);
  for (size_t i = 0; i < inlen; ++i) {
    if (s->c == 128) {
      s->t[0] += s->c;
      if (s->t[0] < s->c) s->t[1]++;
      compress(s, false);
      s->c = 0;
    }
    s->buf[s->c++] = p[i];
  }
}

void blake2b_final(Blake2b* s, void* out) {
  s->t[0] += s->c;
  if (s->t[0] < s->c) s->t[1]++;
  while (s->c < 128) s->buf[s->c++] = 0;
  compress(s, true);
  uint8_t* o = static_cast<uint8_t*>(out);
  for (size_t i = 0; i < s->outlen; ++i) o[i] = static_cast<uint8_t>(s->h[i >> 3] >> (8 * (i & 7)));
}

bool blake2b(void* out, size_t outlen, const void* key, size_t keylen, const void* in, size_t inlen) {
  Blake2b s;
  if (!blake2b_init(&s, outlen, key, keylen)) return false;
  blake2b_update(&s, in, inlen);
  blake2b_final(&s, out);
  return true;
}

}  // namespace pcr

// BLAKE2b (RFC 7693) — chunk keys of the prefix tree (HashPrefix, Alg.1).
#pragma once
#include <cstddef>
#include <cstdint>

namespace pcr {

struct Blake2b {
  uint64_t h[8];
  uint64_t t[2];
  uint8_t buf[128];
  size_t c;
  size_t outlen;
};

// Returns false on bad parameters (outlen not in [1,64] or keylen > 64).
bool blake2b_init(Blake2b* s, size_t outlen, const void* key, size_t keylen);
void blake2b_update(Blake2b* s, const void* in, size_t inlen);
void blake2b_final(Blake2b* s, void* out);
bool blake2b(void* out, size_t outlen, const void* key, size_t keylen, const void* in, size_t inlen);

}  // namespace pcr

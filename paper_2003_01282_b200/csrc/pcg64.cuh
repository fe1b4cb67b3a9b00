// Bit-exact device/host restatement of the reference's probe stream (slq.py:63-72):
//   PCG64(SeedSequence(entropy=seed, spawn_key=(i,))) -> Generator.integers(0, 2, size=n)*2-1
// SeedSequence: numpy's 4-word uint32 hash pool; PCG64: 128-bit LCG with XSL-RR output;
// integers(0,2): bit 31 of each buffered 32-bit half of the 64-bit stream (low half first).
// oracle/pcg64.py is the pure-Python restatement these are tested against.
#pragma once
#include <stdint.h>

#include "../../include/slq_b200.h"

namespace slq {

typedef unsigned __int128 u128;

#define SLQ_HD __host__ __device__ __forceinline__

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

SLQ_HD u128 pcg_mult() {
  return (static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;
}

SLQ_HD uint32_t ss_hash(uint32_t v, uint32_t& c) {
  v ^= c;
  c *= kMultA;
  v *= c;
  return v ^ (v >> 16);
}

SLQ_HD uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> 16);
}

// The seed's run entropy: numpy's SeedSequence takes any non-negative int and splits it into
// little-endian uint32 words (0 -> one zero word).  Up to 8 words (seeds < 2^256) are supported.
constexpr int kSeedWords = 8;
struct SeedKey {
  uint32_t w[kSeedWords];
  int nw;
};

SLQ_HD SeedKey seed_key_u64(uint64_t seed) {
  SeedKey k{};
  k.w[0] = static_cast<uint32_t>(seed);
  k.nw = 1;
  if (seed >> 32) k.w[k.nw++] = static_cast<uint32_t>(seed >> 32);
  return k;
}

// C-ABI seed (slq_b200.h slq_seed) -> SeedKey; false for an invalid word count.
inline bool seed_key_of(const slq_seed* s, SeedKey* out) {
  if (!s || s->nwords < 1 || s->nwords > kSeedWords) return false;
  SeedKey k{};
  for (int i = 0; i < s->nwords; ++i) k.w[i] = s->words[i];
  k.nw = s->nwords;
  *out = k;
  return true;
}

// Entropy words: the seed words (zero-padded to the pool size of 4 because a spawn key is present),
// then the spawn key index as 1-2 words.
SLQ_HD void pcg64_seed_state(const SeedKey& key, uint64_t index, u128* state, u128* inc) {
  uint32_t data[kSeedWords + 2];
  int nd = 0;
  for (int i = 0; i < key.nw && i < kSeedWords; ++i) data[nd++] = key.w[i];
  while (nd < 4) data[nd++] = 0u;
  data[nd++] = static_cast<uint32_t>(index);
  if (index >> 32) data[nd++] = static_cast<uint32_t>(index >> 32);

  uint32_t pool[4];
  uint32_t hc = kInitA;
  for (int i = 0; i < 4; ++i) pool[i] = ss_hash(data[i], hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hash(pool[s], hc));
  for (int s = 4; s < nd; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hash(data[s], hc));

  uint32_t w32[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= kMultB;
    v *= hb;
    w32[i] = v ^ (v >> 16);
  }
  uint64_t w64[4];
  for (int k = 0; k < 4; ++k) w64[k] = static_cast<uint64_t>(w32[2 * k]) | (static_cast<uint64_t>(w32[2 * k + 1]) << 32);
  const u128 initstate = (static_cast<u128>(w64[0]) << 64) | w64[1];
  const u128 initseq = (static_cast<u128>(w64[2]) << 64) | w64[3];
  const u128 mult = pcg_mult();
  u128 incv = (initseq << 1) | 1u;
  u128 st = incv;          // state = 0; step
  st += initstate;
  st = st * mult + incv;   // step
  *state = st;
  *inc = incv;
}

SLQ_HD void pcg64_seed_state(uint64_t seed, uint64_t index, u128* state, u128* inc) {
  pcg64_seed_state(seed_key_u64(seed), index, state, inc);
}

// Advance the LCG by `delta` steps in O(log delta) (Brown's jump-ahead).
SLQ_HD u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1u) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// XSL-RR output of an (already stepped) state.
SLQ_HD uint64_t pcg_output(u128 state) {
  const uint64_t x = static_cast<uint64_t>(state >> 64) ^ static_cast<uint64_t>(state);
  const unsigned rot = static_cast<unsigned>(state >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

}  // namespace slq

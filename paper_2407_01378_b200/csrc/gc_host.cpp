// Host-side helpers of the C ABI: error reporting and the seeding chain.
//
// The reference derives every random stream as
//   splitmix64 chain over (experiment_seed ^ fnv1a64(tag), round, worker + salt)
// (pkg/src/gradcomp/vectors.py:26-39, 64-73) and feeds the result to
// numpy.random.PCG64 (vectors.py:75-76), which seeds through SeedSequence.
// Both numpy algorithms (SeedSequence hashmix pool + generate_state, and the
// pcg64_set_seed / XSL-RR generator) are restated here so the device kernels can
// reproduce the reference's draws without numpy.
#include <cstring>
#include <string>

#include "gc_internal.h"

namespace {
thread_local std::string g_last_error;

constexpr uint64_t kMask32 = 0xFFFFFFFFull;
using u128 = unsigned __int128;
constexpr u128 kPcgMult = (static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;

inline u128 mk(uint64_t hi, uint64_t lo) { return (static_cast<u128>(hi) << 64) | lo; }

// numpy SeedSequence constants (numpy/random/bit_generator.pyx).
constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

struct HashConst {
  uint32_t v;
  uint32_t mix(uint32_t value) {
    value ^= v;
    v *= kMultA;
    value *= v;
    value ^= value >> 16;
    return value;
  }
};

inline uint32_t mix2(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  return r ^ (r >> 16);
}
}  // namespace

void gc_set_error(const std::string &msg) { g_last_error = msg; }

extern "C" {

int gc_version(void) { return GC_ABI_VERSION; }

const char *gc_last_error(void) { return g_last_error.c_str(); }

uint64_t gc_splitmix64(uint64_t value) {
  uint64_t z = value + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t gc_fnv1a64(const char *text, size_t len) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < len; ++i) {
    h ^= static_cast<unsigned char>(text[i]);
    h *= 0x100000001B3ull;
  }
  return h;
}

uint64_t gc_stream_seed(uint64_t experiment_seed, const char *tag, size_t tag_len,
                        uint64_t round_index, int64_t worker) {
  uint64_t h = gc_splitmix64(experiment_seed ^ gc_fnv1a64(tag, tag_len));
  h = gc_splitmix64(h ^ round_index);
  if (worker >= 0) h = gc_splitmix64(h ^ (static_cast<uint64_t>(worker) + 0x517CC1B727220A95ull));
  return h;
}

void gc_pcg64_from_seed(uint64_t seed, gc_pcg64 *out) {
  // SeedSequence(entropy=seed): entropy as little-endian u32 words ([0] for 0).
  uint32_t words[2];
  int nwords = 0;
  if (seed == 0) {
    words[nwords++] = 0;
  } else {
    while (seed) {
      words[nwords++] = static_cast<uint32_t>(seed & kMask32);
      seed >>= 32;
    }
  }
  uint32_t pool[4];
  HashConst hc{kInitA};
  for (int i = 0; i < 4; ++i) pool[i] = hc.mix(i < nwords ? words[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix2(pool[d], hc.mix(pool[s]));
  // (entropy never exceeds the 4-word pool for a 64-bit seed)
  // generate_state(4, uint64): 8 u32 words, paired little-endian.
  uint32_t st[8];
  uint32_t hb = kInitB;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  uint64_t w[4];
  for (int i = 0; i < 4; ++i) w[i] = static_cast<uint64_t>(st[2 * i]) | (static_cast<uint64_t>(st[2 * i + 1]) << 32);
  // pcg64_set_seed: state=0; inc=(initseq<<1)|1; step; state+=initstate; step.
  u128 initstate = mk(w[0], w[1]);
  u128 initseq = mk(w[2], w[3]);
  u128 inc = (initseq << 1) | 1u;
  u128 state = 0;
  state = state * kPcgMult + inc;
  state += initstate;
  state = state * kPcgMult + inc;
  out->state_hi = static_cast<uint64_t>(state >> 64);
  out->state_lo = static_cast<uint64_t>(state);
  out->inc_hi = static_cast<uint64_t>(inc >> 64);
  out->inc_lo = static_cast<uint64_t>(inc);
}

void gc_pcg64_advance(gc_pcg64 *g, uint64_t delta_hi, uint64_t delta_lo) {
  u128 delta = mk(delta_hi, delta_lo);
  u128 inc = mk(g->inc_hi, g->inc_lo);
  u128 cur_mult = kPcgMult, cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1u) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  u128 state = acc_mult * mk(g->state_hi, g->state_lo) + acc_plus;
  g->state_hi = static_cast<uint64_t>(state >> 64);
  g->state_lo = static_cast<uint64_t>(state);
}

uint64_t gc_pcg64_next(gc_pcg64 *g) {
  u128 state = mk(g->state_hi, g->state_lo) * kPcgMult + mk(g->inc_hi, g->inc_lo);
  g->state_hi = static_cast<uint64_t>(state >> 64);
  g->state_lo = static_cast<uint64_t>(state);
  uint64_t x = g->state_hi ^ g->state_lo;
  unsigned rot = static_cast<unsigned>(g->state_hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

}  // extern "C"

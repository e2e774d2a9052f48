// Host-control acceleration: the reference's synthetic
// draft (`/root/reference/pkg/src/treepipe/token_source.py:73-111`) draws every
// proposal from `np.random.default_rng([seed, call_index])`, i.e. a fresh
// SeedSequence-seeded PCG64 per call — ~30 us of numpy per frontier node, the
// bulk of a step's host time at w=64.  This file restates exactly the pieces of
// numpy 2.x that call uses, bit for bit (checked against numpy in
// tests/test_host_control.py over thousands of seeds):
//   SeedSequence(entropy).generate_state(4, uint64)   (pool 4, hashmix/mix)
//   PCG64 (XSL-RR 128/64) seeded with (state, increment) from those words
//   Generator.random()            -> (next64 >> 11) * 2^-53
//   Generator.geometric(p>=1/3)   -> numpy's "search" method
//   Generator.choice(V, size, replace=False)  -> Floyd's algorithm with
//       numpy's open-addressing hash set + _shuffle_int (Lemire bounded
//       32-bit draws on buffered halves of 64-bit outputs)
// and the synthetic_draft logic on top.  Pure host code, no device.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/treepipe_b200.h"

namespace {

// ---- SeedSequence (numpy/random/bit_generator.pyx) --------------------------------
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u;
constexpr int XSHIFT = 16;

struct SeedSeq {
  uint32_t pool[4];
  explicit SeedSeq(const std::vector<uint32_t>& entropy) {
    uint32_t hash_const = INIT_A;
    auto hashmix = [&](uint32_t value) {
      value ^= hash_const;
      hash_const *= MULT_A;
      value *= hash_const;
      value ^= value >> XSHIFT;
      return value;
    };
    auto mix = [](uint32_t x, uint32_t y) {
      uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
      r ^= r >> XSHIFT;
      return r;
    };
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < (int)entropy.size() ? entropy[i] : 0u);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
    for (size_t s = 4; s < entropy.size(); ++s)
      for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(entropy[s]));
  }
  void generate_u64(uint64_t* out, int n64) const {
    uint32_t hash_const = INIT_B;
    std::vector<uint32_t> w(2 * n64);
    for (int i = 0; i < 2 * n64; ++i) {
      uint32_t v = pool[i % 4];
      v ^= hash_const;
      hash_const *= MULT_B;
      v *= hash_const;
      v ^= v >> XSHIFT;
      w[i] = v;
    }
    for (int i = 0; i < n64; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
  }
};

// ---- PCG64 (numpy/random/src/pcg64) ------------------------------------------------
typedef unsigned __int128 u128;
const u128 PCG_MULT = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;

struct Pcg64 {
  u128 state, inc;
  int has_u32 = 0;
  uint32_t u32 = 0;
  Pcg64(const SeedSeq& ss) {
    uint64_t v[4];
    ss.generate_u64(v, 4);
    const u128 initstate = ((u128)v[0] << 64) | v[1];
    const u128 initseq = ((u128)v[2] << 64) | v[3];
    state = 0;
    inc = (initseq << 1) | 1;
    step();
    state += initstate;
    step();
  }
  void step() { state = state * PCG_MULT + inc; }
  uint64_t next64() {
    step();
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  uint32_t next32() {
    if (has_u32) {
      has_u32 = 0;
      return u32;
    }
    const uint64_t n = next64();
    has_u32 = 1;
    u32 = (uint32_t)(n >> 32);
    return (uint32_t)(n & 0xffffffffu);
  }
  double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
  // random_bounded_uint64(off=0, rng, mask=0, use_masked=0) for rng < 2^32 - 1
  uint64_t bounded(uint64_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFull) return next32();
    const uint32_t rng_excl = (uint32_t)rng + 1;
    uint64_t m = (uint64_t)next32() * rng_excl;
    uint32_t leftover = (uint32_t)(m & 0xFFFFFFFFull);
    if (leftover < rng_excl) {
      const uint32_t threshold = (uint32_t)((0xFFFFFFFFu - (uint32_t)rng) % rng_excl);
      while (leftover < threshold) {
        m = (uint64_t)next32() * rng_excl;
        leftover = (uint32_t)(m & 0xFFFFFFFFull);
      }
    }
    return m >> 32;
  }
};

// Generator.choice(pop, size, replace=False, shuffle=True), Floyd branch.
bool choice_floyd(Pcg64& g, int64_t pop, int64_t size, int64_t* idx) {
  if (pop > 10000 && size > pop / 50) return false;  // numpy's tail-shuffle branch: not restated
  uint64_t mask = (uint64_t)(1.2 * (double)size);
  for (int s = 1; s <= 32; s <<= 1) mask |= mask >> s;
  std::vector<uint64_t> hs(mask + 1, ~0ull);
  for (int64_t j = pop - size; j < pop; ++j) {
    const uint64_t val = g.bounded((uint64_t)j);
    uint64_t loc = val & mask;
    while (hs[loc] != ~0ull && hs[loc] != val) loc = (loc + 1) & mask;
    if (hs[loc] == ~0ull) {
      hs[loc] = val;
      idx[j - pop + size] = (int64_t)val;
    } else {
      loc = (uint64_t)j & mask;
      while (hs[loc] != ~0ull) loc = (loc + 1) & mask;
      hs[loc] = (uint64_t)j;
      idx[j - pop + size] = j;
    }
  }
  for (int64_t i = size - 1; i >= 1; --i) {  // _shuffle_int(size, first=1)
    const uint64_t j = g.bounded((uint64_t)i);
    std::swap(idx[j], idx[i]);
  }
  return true;
}

std::vector<uint32_t> entropy_words(uint64_t seed, int64_t index) {
  std::vector<uint32_t> out;
  for (uint64_t v : {seed, (uint64_t)index}) {
    if (v == 0) {
      out.push_back(0u);
      continue;
    }
    while (v) {
      out.push_back((uint32_t)(v & 0xffffffffu));
      v >>= 32;
    }
  }
  return out;
}

}  // namespace

extern "C" {

// One synthetic_draft call (token_source.py:73-111): tokens_out[0..*n_out).
// oracle_next < 0 means "no bound continuation".  Returns TP_ECONFIG when the
// call would take a numpy branch this restatement does not cover (the caller
// then falls back to numpy): geometric with p < 1/3, or the tail-shuffle
// choice branch.
int tp_synthetic_draft(uint64_t seed, int64_t call_index, int32_t oracle_next, double top1_hit, double rank_decay,
                       double miss_prob, int32_t k, int32_t vocab, int32_t* tokens_out, int32_t* n_out) {
  if (k < 1 || vocab < 1) return TP_ESHAPE;
  Pcg64 g{SeedSeq(entropy_words(seed, call_index))};
  int truth_rank = 0;  // 0 = absent
  if (oracle_next >= 0) {
    const double u = g.next_double();
    if (u >= miss_prob) {
      if (u < miss_prob + top1_hit) {
        truth_rank = 1;
      } else if (rank_decay == 0.0) {
        truth_rank = 2;
      } else {
        const double p = 1.0 - rank_decay;
        if (!(p >= 0.333333333333333333333333)) return TP_ECONFIG;
        int64_t x = 1;
        double sum = p, prod = p;
        const double q = 1.0 - p;
        const double U = g.next_double();
        while (U > sum) {
          prod *= q;
          sum += prod;
          ++x;
        }
        truth_rank = (int)(1 + x);
        if (truth_rank > k) truth_rank = 0;
      }
    }
  }
  const int64_t size = std::min<int64_t>(vocab, (int64_t)k + 1);
  std::vector<int64_t> draws(size);
  if (!choice_floyd(g, vocab, size, draws.data())) return TP_ECONFIG;
  std::vector<int32_t> pool;
  pool.reserve(size);
  for (int64_t t : draws)
    if (oracle_next < 0 || t != oracle_next) pool.push_back((int32_t)t);
  const int take = (int)std::min<int64_t>(k, (int64_t)pool.size() + (truth_rank ? 1 : 0));
  size_t it = 0;
  for (int slot = 0; slot < take; ++slot) {
    if (truth_rank && slot == truth_rank - 1) {
      tokens_out[slot] = oracle_next;
    } else {
      if (it >= pool.size()) return TP_ECONFIG;  // the reference raises StopIteration here: let numpy do it
      tokens_out[slot] = pool[it++];
    }
  }
  *n_out = take;
  return TP_OK;
}

// `count` consecutive calls (call_index0 + i) in one go; tokens_out is [count][k].
int tp_synthetic_draft_batch(int32_t count, uint64_t seed, int64_t call_index0, const int32_t* oracle_next,
                             double top1_hit, double rank_decay, double miss_prob, int32_t k, int32_t vocab,
                             int32_t* tokens_out, int32_t* n_out) {
  for (int i = 0; i < count; ++i) {
    const int rc = tp_synthetic_draft(seed, call_index0 + i, oracle_next[i], top1_hit, rank_decay, miss_prob, k,
                                      vocab, tokens_out + (size_t)i * k, n_out + i);
    if (rc != TP_OK) return rc;
  }
  return TP_OK;
}

}  // extern "C"

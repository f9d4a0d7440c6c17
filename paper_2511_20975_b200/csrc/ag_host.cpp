// Host-side input synthesis: the reference's accuracy-label generator
// (generate_accurate_set, src/accuracy.cpp:144-198) so benches and callers
// can build AccurateSet batches without the reference.  Off the hot path:
// it only produces the seed/removed CSR that the GPU kernels consume.
#include <cmath>
#include <cstring>
#include <vector>

#include "ag_internal.h"

using agb::fail;

namespace {

// rng::Stream draws (rng.h:64-96) over a bare state word.
// splitmix64 with state advance, exactly rng::splitmix64 (rng.h:34-39)
inline uint64_t next_u64(uint64_t& state) {
  state += agb::kGamma;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline double next_unit(uint64_t& st) { return (double)(next_u64(st) >> 11) * 0x1.0p-53; }
inline uint64_t next_below(uint64_t& st, uint64_t n) { return next_u64(st) % n; }
inline bool bernoulli(uint64_t& st, double p) { return next_unit(st) < p; }

inline uint64_t mix(std::initializer_list<uint64_t> w) {
  uint64_t s = agb::kMixIV;
  for (uint64_t x : w) s = agb::absorb(s, x);
  return s;
}

using Cfg = std::vector<uint8_t>;

// compare_configs (workflow.cpp:189-202): 0 eq, 1 below, 2 above, 3 incomparable
int cmp(const Cfg& x, const Cfg& y) {
  bool le = true, ge = true;
  for (size_t i = 0; i < x.size(); ++i) {
    if (x[i] > y[i]) le = false;
    if (x[i] < y[i]) ge = false;
  }
  return le && ge ? 0 : le ? 1 : ge ? 2 : 3;
}

uint64_t encode(const Cfg& c, int m) {
  uint64_t idx = 0;
  for (uint8_t d : c) idx = idx * (uint64_t)m + d;
  return idx;
}

void decode(uint64_t idx, int n, int m, Cfg& c) {
  c.resize(n);
  for (int i = n - 1; i >= 0; --i) {
    c[i] = (uint8_t)(idx % (uint64_t)m);
    idx /= (uint64_t)m;
  }
}

bool contains(const std::vector<Cfg>& seeds, const Cfg& c) {
  for (const Cfg& s : seeds)
    if (cmp(s, c) <= 1) return true;
  return false;
}

// net violation change if c were removed (accuracy.cpp:65-82)
long long removal_delta(int m, const std::vector<char>& member, Cfg& c) {
  long long delta = 0;
  for (size_t i = 0; i < c.size(); ++i) {
    if (c[i] > 0) {
      --c[i];
      if (member[encode(c, m)]) ++delta;
      ++c[i];
    }
    if (c[i] + 1 < m) {
      ++c[i];
      if (!member[encode(c, m)]) --delta;
      --c[i];
    }
  }
  return delta;
}

}  // namespace

extern "C" int ag_generate_truth(const ag_space* space, const ag_gen_params* p, uint64_t seed,
                                 uint64_t salt, uint64_t first_id, int32_t count,
                                 int32_t* seed_ptr, uint8_t* seeds_out, int32_t seeds_cap,
                                 int32_t* removed_ptr, uint64_t* removed_out,
                                 int32_t removed_cap) {
  if (!space || !p) return fail(AG_ERR_VALIDATION, "null argument");
  // AccuracyGenParams::validate (accuracy.cpp:126-142)
  if (p->p_easy < 0 || p->p_medium < 0 || p->p_hard < 0 ||
      p->p_easy + p->p_medium + p->p_hard <= 0)
    return fail(AG_ERR_VALIDATION, "difficulty mix needs nonnegative weights, sum > 0");
  if (p->easy_base_prob < 0 || p->easy_base_prob > 1)
    return fail(AG_ERR_VALIDATION, "easy_base_prob outside [0, 1]");
  if (p->violation_rate < 0 || p->violation_rate >= 1)
    return fail(AG_ERR_VALIDATION, "violation_rate outside [0, 1)");
  const int n = space->n, m = space->m;
  const uint64_t size = space->size;
  if (p->violation_rate > 0 && (size == 0 || size > 4096))
    return fail(AG_ERR_VALIDATION, "violation injection needs an enumerable configuration space");

  int32_t rows = 0, nrem = 0;
  seed_ptr[0] = 0;
  removed_ptr[0] = 0;
  for (int32_t q = 0; q < count; ++q) {
    uint64_t st = mix({seed, salt, first_id + (uint64_t)q});
    const double total = p->p_easy + p->p_medium + p->p_hard;
    const double u = next_unit(st) * total;
    std::vector<Cfg> seeds;
    if (u < p->p_easy) {
      if (bernoulli(st, p->easy_base_prob)) {
        seeds.push_back(Cfg(n, 0));
      } else {
        size_t k = 1 + next_below(st, 2);
        for (size_t s = 0; s < k; ++s) {
          Cfg c(n, 0);
          bool base = true;
          for (int i = 0; i < n; ++i) {
            double v = next_unit(st);
            int d = (int)(v * v * m);
            c[i] = (uint8_t)(d < m - 1 ? d : m - 1);
            base &= c[i] == 0;
          }
          if (base) c[next_below(st, (uint64_t)n)] = 1;
          seeds.push_back(c);
        }
      }
    } else if (u < p->p_easy + p->p_medium) {
      size_t k = 1 + next_below(st, 2);
      for (size_t s = 0; s < k; ++s) {
        Cfg c(n);
        for (int i = 0; i < n; ++i) c[i] = (uint8_t)next_below(st, (uint64_t)m);
        seeds.push_back(c);
      }
    } else {
      seeds.push_back(Cfg(n, (uint8_t)(m - 1)));
    }
    // minimalize (accuracy.cpp:28-42)
    std::vector<Cfg> kept;
    for (size_t i = 0; i < seeds.size(); ++i) {
      bool dominated = false;
      for (size_t j = 0; j < seeds.size() && !dominated; ++j) {
        if (i == j) continue;
        int o = cmp(seeds[j], seeds[i]);
        if (o == 1 || (o == 0 && j < i)) dominated = true;
      }
      if (!dominated) kept.push_back(seeds[i]);
    }
    if (rows + (int32_t)kept.size() > seeds_cap) return fail(AG_ERR_VALIDATION, "seeds_cap too small");
    for (const Cfg& c : kept) std::memcpy(seeds_out + (size_t)(rows++) * n, c.data(), n);
    seed_ptr[q + 1] = rows;

    if (p->violation_rate > 0) {  // inject_violations (accuracy.cpp:84-112)
      uint64_t edges = (uint64_t)(m - 1) * (size / (uint64_t)m) * (uint64_t)n;
      double expectation = p->violation_rate * (double)edges;
      uint64_t target = (uint64_t)std::floor(expectation);
      if (bernoulli(st, expectation - std::floor(expectation))) ++target;
      if (target > 0) {
        std::vector<char> member(size);
        Cfg c;
        for (uint64_t i = 0; i < size; ++i) {
          decode(i, n, m, c);
          member[i] = contains(kept, c);
        }
        uint64_t violated = 0;
        std::vector<uint64_t> cand;
        while (violated < target) {
          uint64_t remaining = target - violated;
          cand.clear();
          for (uint64_t i = 0; i < size; ++i) {
            if (!member[i] || i == size - 1) continue;
            decode(i, n, m, c);
            long long d = removal_delta(m, member, c);
            if (d >= 1 && (uint64_t)d <= remaining) cand.push_back(i);
          }
          if (cand.empty()) break;
          uint64_t pick = cand[next_below(st, cand.size())];
          decode(pick, n, m, c);
          violated += (uint64_t)removal_delta(m, member, c);
          member[pick] = 0;
          if (nrem >= removed_cap) return fail(AG_ERR_VALIDATION, "removed_cap too small");
          removed_out[nrem++] = pick;
        }
      }
    }
    removed_ptr[q + 1] = nrem;
  }
  return AG_OK;
}

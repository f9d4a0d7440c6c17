// Routing hot path, enumerate mode (K1 score -> K2 scans -> K3 compact).
//
// Replaces the exhaustive scoring loop of enumerate_members
// (reference src/accuracy.cpp:227-238) / oracle_accurate_set
// (tests/acceptance/criteria.cpp:93-101) driven through
// RouterBackend::evaluate (include/aragog/router.h:33-41).
//
// Work decomposition: a warp-task is up to 1024 consecutive 32-index bitmap
// words (32K canonical indices) of one request; each of its 32 iterations
// gives one word to each lane.  Nothing is read per configuration: the
// configuration is the index.  HBM traffic is the output only (1/8 B per
// config of bitmap, 4 B per member).
//
// Verdict per configuration c (digits d[0..N-1], position 0 most significant):
//   truth(c)  = c not in removed  &&  exists seed s <= c pointwise
//             (AccurateSet::contains, accuracy.cpp:116-124)
//   Write c = (Q, x, l): Q = digits 0..N-3, x = digit N-2, l = digit N-1.
//   Inside one word l(j) = (l0 + j) mod M for every position j, and (Q, x)
//   change only at row / block boundaries.  A seed s with s.Q <= Q
//   contributes the positions with x(j) >= s.x (a suffix of the segment) and
//   l(j) >= s.l (a periodic mask, tabulated once per space): a word costs
//   O(#seeds) mask operations instead of O(32 * N) compares.  s.Q <= Q runs
//   SWAR on packed bytes: ((Q | H) - s.Q) & H == H (all digits < 128).
//   noisy(c)  = truth ? k >= t_fn : k < t_fp, k = mix({seed, 0xA3, id,
//             hash_config(c)}) >> 11 (router.cpp:22-28,50-57); the hash chain
//             is tabulated per space (hash_config is request-independent),
//             so a scored configuration costs one splitmix64 over a
//             coalesced table load, lane = bit; only words holding a bit the
//             noise can change are visited (generic path: the chain carried
//             incrementally, two finalisers per configuration).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "ag_internal.h"

namespace agb {

namespace {

#ifndef AG_ROUTE_WARPS
#define AG_ROUTE_WARPS 8
#endif
constexpr int kWarpsPerBlock = AG_ROUTE_WARPS;
constexpr int kThreads = kWarpsPerBlock * 32;
constexpr int kMaxFastSeeds = 32;    // per-warp packed-seed cache
constexpr uint32_t kTaskIters = 32;  // iterations of 32 words per warp-task
constexpr uint32_t kTaskWords = 32 * kTaskIters;

template <int NT>
struct DigitsT {
  static constexpr int kN = NT > 0 ? NT : kMaxAgents;
};

// thr(row) with per-digit compares (any N <= 32, any M): generic fallback.
template <int NT>
__device__ __forceinline__ uint32_t row_threshold(const uint32_t (&d)[DigitsT<NT>::kN], int n,
                                                  const uint8_t* __restrict__ seeds, int k,
                                                  uint32_t m) {
  constexpr int kN = DigitsT<NT>::kN;
  const int nn = NT > 0 ? NT : n;
  uint32_t thr = m;
  for (int s = 0; s < k; ++s) {
    const uint8_t* sd = seeds + (size_t)s * nn;
    bool ok = true;
#pragma unroll
    for (int a = 0; a < kN - 1; ++a) {
      if (NT == 0 && a >= nn - 1) break;
      ok &= (uint32_t)__ldg(sd + a) <= d[a];
    }
    const uint32_t last = __ldg(sd + nn - 1);
    if (ok && last < thr) thr = last;
  }
  return thr;
}

// digits of x (workflow.cpp:263-275)
template <int NT>
__device__ __forceinline__ void decode(const SpaceDev& sp, uint32_t x,
                                       uint32_t (&d)[DigitsT<NT>::kN]) {
  constexpr int kN = DigitsT<NT>::kN;
  const int n = NT > 0 ? NT : sp.n;
  const uint32_t m = (uint32_t)sp.m;
#pragma unroll
  for (int a = kN - 1; a >= 0; --a) {
    if (NT == 0 && a >= n) continue;
    const uint32_t q = divm(x, sp.div_m);
    d[a] = x - q * m;
    x = q;
  }
}

// bits [lo, hi) of a 32-bit word, lo/hi clipped to [0, 32]
__device__ __forceinline__ uint32_t range_bits(int lo, int hi) {
  lo = max(lo, 0);
  hi = min(hi, 32);
  if (lo >= hi) return 0u;
  return (uint32_t)(((1ull << hi) - 1ull) & ~((1ull << lo) - 1ull));
}

// Truth word, generic path (row by row).
template <int NT>
__device__ __forceinline__ uint32_t truth_word_generic(const SpaceDev& sp, uint32_t i0,
                                                       uint32_t nbits,
                                                       const uint8_t* __restrict__ seeds, int k) {
  constexpr int kN = DigitsT<NT>::kN;
  const int n = NT > 0 ? NT : sp.n;
  const uint32_t m = (uint32_t)sp.m;
  uint32_t d[kN];
  decode<NT>(sp, i0, d);
  int pos = -(int)d[n - 1];
  uint32_t bits = 0;
  while (pos < (int)nbits) {
    const uint32_t thr = row_threshold<NT>(d, n, seeds, k, m);
    bits |= range_bits(pos + (int)thr, pos + (int)m);
    pos += (int)m;
    bool carry = true;  // next row: increment digits 0..N-2
#pragma unroll
    for (int a = kN - 2; a >= 0; --a) {
      if (NT == 0 && a >= n - 1) continue;
      if (carry) {
        if (++d[a] == m) d[a] = 0;
        else carry = false;
      }
    }
  }
  return bits & range_bits(0, (int)nbits);
}

// Per-warp packed seeds for the 2-D mask path.
struct PackedSeeds {
  uint64_t q[kMaxFastSeeds];  // digits 0..N-3, byte b = digit N-3-b
  uint32_t xl[kMaxFastSeeds]; // digit N-2 in bits 8..15, digit N-1 in bits 0..7
};

// Digit state of a word start i0 = ((Q * M) + x) * M + l0 for the 2-D path:
// Q packed as bytes (byte b = digit N-3-b).  Carried from word to word so
// the hot loop never divides.
struct WordPos {
  uint32_t l0, x;
  uint64_t Q;
};

__device__ __forceinline__ WordPos word_pos(const SpaceDev& sp, uint32_t i0) {
  const uint32_t m = (uint32_t)sp.m;
  WordPos p;
  const uint32_t y = divm(i0, sp.div_m);
  p.l0 = i0 - y * m;
  uint32_t v = divm(y, sp.div_m);
  p.x = y - v * m;
  p.Q = 0;
  for (int b = 0; b < sp.n - 2; ++b) {
    const uint32_t v2 = divm(v, sp.div_m);
    p.Q |= (uint64_t)(v - v2 * m) << (8 * b);
    v = v2;
  }
  return p;
}

// add `inc` (< 128) to the packed block number, propagating carries
__device__ __forceinline__ uint64_t q_add(uint64_t Q, uint32_t inc, uint32_t m, int nq) {
  Q += inc;
  for (int b = 0; b < nq; ++b) {
    const uint32_t v = (uint32_t)(Q >> (8 * b)) & 0xFFu;
    if (v < m) break;
    const uint32_t carry = v / m;
    Q -= (uint64_t)(carry * m) << (8 * b);
    if (b + 1 < 8) Q += (uint64_t)carry << (8 * (b + 1));
  }
  return Q;
}

// advance a word position by 32 indices (M <= 32); divisions by M use the
// precomputed 64-bit reciprocal
__device__ __forceinline__ void advance32(WordPos& p, uint32_t m, uint64_t div_m, int nq) {
  const uint32_t l = p.l0 + 32;
  const uint32_t rows = divm(l, div_m);
  p.l0 = l - rows * m;
  const uint32_t xs = p.x + rows;
  if (xs >= m) {
    const uint32_t blocks = divm(xs, div_m);
    p.x = xs - blocks * m;
    p.Q = q_add(p.Q, blocks, m, nq);
  } else {
    p.x = xs;
  }
}

// Truth word, 2-D mask path (2 <= N <= 10, M <= 32).
__device__ __forceinline__ uint32_t truth_word_2d(WordPos p, uint32_t m, int nq, uint32_t nbits,
                                                  const PackedSeeds& ps, int k, uint64_t H,
                                                  const uint32_t* __restrict__ colmask) {
  const uint32_t* cm = colmask + p.l0 * 32;  // colmask[l0][c]
  uint32_t bits = 0;
  int j0 = 0;
  int ls = (int)p.l0;  // last digit at j0
  uint32_t x = p.x;
  uint64_t Q = p.Q;
  while (j0 < (int)nbits) {
    // segment [j0, j1): rows x .. M-1 of block Q
    const int rowstart = j0 - ls;  // position of the first row's start
    const int j1 = min((int)nbits, rowstart + (int)(m - x) * (int)m);
    for (int s = 0; s < k; ++s) {
      if (((((Q | H) - ps.q[s]) & H) == H)) {
        const uint32_t sx = ps.xl[s] >> 8, sl = ps.xl[s] & 0xFFu;
        const int jx = sx > x ? rowstart + (int)(sx - x) * (int)m : j0;
        bits |= __ldg(cm + sl) & range_bits(jx, j1);
      }
    }
    // next block: Q + 1, x = 0, last digit 0
    j0 = j1;
    ls = 0;
    x = 0;
    Q = q_add(Q, 1, m, nq);
  }
  return bits & range_bits(0, (int)nbits);
}

// Noise pass over a truth word: re-verdicts every configuration whose verdict
// the router noise can change (router.cpp:50-57).
template <int NT>
__device__ __forceinline__ uint32_t noisy_word(const SpaceDev& sp, uint32_t i0, uint32_t nbits,
                                               uint32_t truth, const RouterDev& rt, uint64_t P) {
  constexpr int kN = DigitsT<NT>::kN;
  const int n = NT > 0 ? NT : sp.n;
  const uint32_t m = (uint32_t)sp.m;
  const uint32_t valid = range_bits(0, (int)nbits);
  const uint32_t need = ((rt.t_fn > 0) ? truth : 0u) | ((rt.t_fp > 0) ? ~truth : 0u);
  uint32_t out = truth & ~need;
  if (!(need & valid)) return out & valid;
  uint32_t d[kN];
  decode<NT>(sp, i0, d);
  uint64_t h[kN];  // h[a] = hash after digits 0..a-1, valid for a < hvalid
  h[0] = kHashIV;
  int hvalid = 1;
  uint64_t s1 = 0;
  bool s1_ok = false;
  uint32_t dl = d[n - 1];
  for (uint32_t j = 0; j < nbits; ++j) {
    if ((need >> j) & 1u) {
      if (!s1_ok) {
#pragma unroll
        for (int a = 0; a < kN - 1; ++a) {
          if (NT == 0 && a >= n - 1) break;
          if (a + 1 >= hvalid) h[a + 1] = absorb(absorb(kMixIV, h[a]), d[a]);
        }
        hvalid = n;
        s1 = absorb(kMixIV, h[n - 1]);
        s1_ok = true;
      }
      const uint64_t key = absorb(P, absorb(s1, dl)) >> 11;
      const bool t = (truth >> j) & 1u;
      const bool v = t ? key >= rt.t_fn : key < rt.t_fp;
      out |= (uint32_t)v << j;
    }
    if (++dl == m) {
      dl = 0;
      if (j + 1 < nbits) {
        int changed = n - 1;
        bool carry = true;
#pragma unroll
        for (int a = kN - 2; a >= 0; --a) {
          if (NT == 0 && a >= n - 1) continue;
          if (carry) {
            changed = a;
            if (++d[a] == m) d[a] = 0;
            else carry = false;
          }
        }
        if (changed + 1 < hvalid) hvalid = changed + 1;
        s1_ok = false;
      }
    }
  }
  return out & valid;
}

struct ScoreArgs {
  SpaceDev sp;
  TruthDev t;
  RouterDev rt;
  uint64_t begin, end;
  uint32_t W;        // words per request
  uint32_t C;        // warp-tasks per request
  uint64_t div_c;    // ceil(2^64 / C)
  int R;
  uint32_t flags;
  uint64_t H;        // SWAR high-bit mask over N-2 bytes
  int path2d;        // 2-D mask path available for this space
  int pat_lg;        // phase-pattern path: log2 gcd(M*M, 32), -1 = unavailable
  int pat_P;         // phases per block (M*M / gcd)
  const uint32_t* colmask;
  const uint64_t* hc;  // hash_config(c) per canonical index (noisy router), or null
  uint32_t* bitmap;  // [R * W]
  uint32_t* task_counts;
  // C == 1 (a task is a whole request): the group scan (K2a) fused into the
  // scoring kernel -- group offsets and the request's count written here
  int fuse_scan;
  uint64_t* task_off;
  uint64_t* counts;
};

// Phase-pattern path (M*M >= 32 and few phases): a 32-index word starting at
// block offset o (block = the M*M indices sharing digits 0..N-3) holds the
// same (x, l) digit pattern for every block, so the verdict word of a seed s
// is lo(s, o) when s.Q <= Q plus hi(s, o) when s.Q <= Q + 1 (the part of the
// word that runs into the next block).  Offsets of the words of a request
// form P = M*M / gcd(M*M, 32) phases, tabulated per warp-task once; a word
// then costs two SWAR prefix tests and two ORs per seed.
constexpr int kPatSeeds = 4;
constexpr int kPatMax = 32;

union PatTable {
  struct {
    uint32_t lo[kPatSeeds][kPatMax];
    uint32_t hi[kPatSeeds][kPatMax];
  };
  // up to two seeds (what the generator emits), rebuilt in place: the OR of
  // the seeds' words for every subset of seeds whose prefix test passes,
  // [phase][subset]
  struct {
    uint32_t clo[kPatMax][4];
    uint32_t chi[kPatMax][4];
  };
};

template <int NT>
__global__ void __launch_bounds__(kThreads) k_route_score(ScoreArgs a) {
  __shared__ PackedSeeds s_seeds[kWarpsPerBlock];
  __shared__ uint32_t s_tr[kWarpsPerBlock][32][33];
  __shared__ PatTable s_pat[kWarpsPerBlock];  // phase tables (truth words)
  // the scan / compaction kernels may launch now and wait for this grid
  // (programmatic dependent launch): their launch latency overlaps K1
  asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t task = blockIdx.x * kWarpsPerBlock + wid;
  if ((uint64_t)task >= (uint64_t)a.R * a.C) return;
  // exact task / C (ceil(2^64/C) magic; C == 1 has no 64-bit magic)
  const uint32_t r = a.C == 1 ? task : (uint32_t)__umul64hi(task, a.div_c);
  const uint32_t c = task - r * a.C;
  const int n = NT > 0 ? NT : a.sp.n;
  const int s0 = __ldg(a.t.seed_ptr + r), s1 = __ldg(a.t.seed_ptr + r + 1);
  const int k = s1 - s0;
  const uint8_t* seeds = a.t.seeds + (size_t)s0 * n;
  const bool fast = a.path2d && k <= kMaxFastSeeds;
  if (fast) {
    if (lane < k) {
      const uint8_t* sd = seeds + (size_t)lane * n;
      uint64_t q = 0;
      for (int b = 0; b < n - 2; ++b) q |= (uint64_t)__ldg(sd + n - 3 - b) << (8 * b);
      s_seeds[wid].q[lane] = q;
      s_seeds[wid].xl[lane] = ((uint32_t)__ldg(sd + n - 2) << 8) | __ldg(sd + n - 1);
    }
    __syncwarp();
  }
  const int r0 = __ldg(a.t.removed_ptr + r), r1 = __ldg(a.t.removed_ptr + r + 1);
  uint64_t P = 0;
  if (a.rt.kind == AG_ROUTER_NOISY)
    P = absorb(absorb(absorb(kMixIV, a.rt.noise_seed), kRouterSalt), __ldg(a.t.request_ids + r));
  const uint64_t top = a.sp.size - 1;
  const uint32_t m = (uint32_t)a.sp.m;
  const int nq = a.sp.n - 2;
  uint32_t cnt = 0;
  // lane L owns the 32 consecutive words wbeg + 32L .. +31 (digit state is
  // carried, no division per word); words go through a padded shared-memory
  // transpose so the bitmap stores stay coalesced.
  const uint32_t wbeg = c * kTaskWords;
  const uint32_t wend = min(a.W, wbeg + kTaskWords);
  const uint32_t wl = wbeg + 32u * lane;
  const uint32_t i0s = (uint32_t)(a.begin + (uint64_t)wl * 32);  // < 2^32 when wl < wend
  // all 32 words of this lane are full and inside [begin, end)
  const bool full = (uint64_t)i0s + 1024 <= a.end && wl + 32 <= wend;
  // noisy verdicts deferred to a word-parallel pass when the
  // per-configuration hash is tabulated
  const bool defer = a.rt.kind == AG_ROUTER_NOISY && a.hc != nullptr;
  const bool extras = (r1 > r0) || (a.rt.kind == AG_ROUTER_NOISY && !defer) ||
                      ((a.flags & AG_FORCE_TOP) && !defer);
  const bool pat = fast && !extras && a.pat_lg >= 0 && k <= kPatSeeds;
  if (pat) {
    // phase tables of this task's seeds: lanes own (seed, phase) entries
    const uint32_t Bq = m * m, g = 1u << a.pat_lg;
    const uint32_t r0 = (uint32_t)(a.begin % g);  // every word offset is = r0 (mod g)
    // one (seed, phase) entry per pass, lane = bit position
    for (int s = 0; s < k; ++s) {
      const uint32_t sx = s_seeds[wid].xl[s] >> 8, sl = s_seeds[wid].xl[s] & 0xFFu;
      for (int p = 0; p < a.pat_P; ++p) {
        uint32_t t = r0 + g * (uint32_t)p + (uint32_t)lane;
        const bool nxt = t >= Bq;
        if (nxt) t -= Bq;
        const uint32_t x = divm(t, a.sp.div_m), l = t - x * m;
        const bool in = x >= sx && l >= sl;
        const uint32_t lo = __ballot_sync(0xffffffffu, in && !nxt);
        const uint32_t hi = __ballot_sync(0xffffffffu, in && nxt);
        if (lane == 0) {
          s_pat[wid].lo[s][p] = lo;
          s_pat[wid].hi[s][p] = hi;
        }
      }
    }
    __syncwarp();
    if (k <= 2) {
      PatTable& pt = s_pat[wid];
      const bool own = lane < a.pat_P;
      const uint32_t l0 = own && k > 0 ? pt.lo[0][lane] : 0u, l1 = own && k > 1 ? pt.lo[1][lane] : 0u;
      const uint32_t h0 = own && k > 0 ? pt.hi[0][lane] : 0u, h1 = own && k > 1 ? pt.hi[1][lane] : 0u;
      __syncwarp();  // the per-seed rows are read before the combinations overwrite them
      pt.clo[lane][0] = 0u;
      pt.clo[lane][1] = l0;
      pt.clo[lane][2] = l1;
      pt.clo[lane][3] = l0 | l1;
      pt.chi[lane][0] = 0u;
      pt.chi[lane][1] = h0;
      pt.chi[lane][2] = h1;
      pt.chi[lane][3] = h0 | h1;
    }
    __syncwarp();
  }
  if (pat && full && k <= 2) {
    // hot path, at most two seeds: the prefix tests change only when the
    // word crosses into the next block, so a word is two table loads
    const WordPos p0 = word_pos(a.sp, i0s);
    const uint32_t Bq = m * m;
    uint32_t o = p0.x * m + p0.l0;
    uint64_t Qn = q_add(p0.Q, 1, m, nq);
    const int lg = a.pat_lg;
    const PatTable& pt = s_pat[wid];
    const uint64_t sq0 = k > 0 ? s_seeds[wid].q[0] : ~0ull, sq1 = k > 1 ? s_seeds[wid].q[1] : ~0ull;
    auto tests = [&](uint64_t Q) -> uint32_t {  // bit s: every digit of Q >= seed s's
      return (k > 0 && (((Q | a.H) - sq0) & a.H) == a.H ? 1u : 0u) |
             (k > 1 && (((Q | a.H) - sq1) & a.H) == a.H ? 2u : 0u);
    };
    uint32_t mlo = tests(p0.Q), mhi = tests(Qn);
#pragma unroll 4
    for (uint32_t it = 0; it < 32; ++it) {
      const uint32_t ph = o >> lg;
      const uint32_t word = pt.clo[ph][mlo] | pt.chi[ph][mhi];
      o += 32;
      if (o >= Bq) {
        o -= Bq;
        Qn = q_add(Qn, 1, m, nq);
        mlo = mhi;
        mhi = tests(Qn);
      }
      cnt += __popc(word);
      s_tr[wid][lane][it] = word;
    }
  } else if (pat && full) {
    // hot path: oracle router, no removals, 32 full words, phase tables
    const WordPos p0 = word_pos(a.sp, i0s);
    const uint32_t Bq = m * m;
    uint32_t o = p0.x * m + p0.l0;
    uint64_t Q = p0.Q, Qn = q_add(p0.Q, 1, m, nq);
    const int lg = a.pat_lg;
    const PatTable& pt = s_pat[wid];
    uint64_t sq[kPatSeeds];
#pragma unroll
    for (int s = 0; s < kPatSeeds; ++s) sq[s] = s < k ? s_seeds[wid].q[s] : ~0ull;
#pragma unroll 4
    for (uint32_t it = 0; it < 32; ++it) {
      const uint32_t ph = o >> lg;
      uint32_t word = 0;
#pragma unroll
      for (int s = 0; s < kPatSeeds; ++s) {
        if (s < k) {
          if ((((Q | a.H) - sq[s]) & a.H) == a.H) word |= pt.lo[s][ph];
          if ((((Qn | a.H) - sq[s]) & a.H) == a.H) word |= pt.hi[s][ph];
        }
      }
      o += 32;
      if (o >= Bq) {
        o -= Bq;
        Q = Qn;
        Qn = q_add(Qn, 1, m, nq);
      }
      cnt += __popc(word);
      s_tr[wid][lane][it] = word;
    }
  } else if (fast && full && !extras) {
    // hot path: oracle router, no removals, 32 full words
    WordPos pos = word_pos(a.sp, i0s);
#pragma unroll 4
    for (uint32_t it = 0; it < 32; ++it) {
      const uint32_t word = truth_word_2d(pos, m, nq, 32u, s_seeds[wid], k, a.H, a.colmask);
      advance32(pos, m, a.sp.div_m, nq);
      cnt += __popc(word);
      s_tr[wid][lane][it] = word;
    }
  } else {
    WordPos pos{};
    if (fast && wl < wend) pos = word_pos(a.sp, i0s);
    uint64_t i0 = a.begin + (uint64_t)wl * 32;
    for (uint32_t it = 0; it < 32; ++it, i0 += 32) {
      const uint32_t w = wl + it;
      uint32_t word = 0;
      if (w < wend) {
        const uint32_t nbits = (uint32_t)min((uint64_t)32, a.end - i0);
        if (fast) {
          word = truth_word_2d(pos, m, nq, nbits, s_seeds[wid], k, a.H, a.colmask);
          advance32(pos, m, a.sp.div_m, nq);
        } else {
          word = truth_word_generic<NT>(a.sp, (uint32_t)i0, nbits, seeds, k);
        }
        // removed configurations (AccurateSet::removed, accuracy.cpp:117-119)
        for (int i = r0; i < r1; ++i) {
          const uint64_t x = __ldg(a.t.removed + i);
          if (x >= i0 && x < i0 + nbits) word &= ~(1u << (uint32_t)(x - i0));
        }
        if (a.rt.kind == AG_ROUTER_NOISY && !defer)
          word = noisy_word<NT>(a.sp, (uint32_t)i0, nbits, word, a.rt, P);
        if ((a.flags & AG_FORCE_TOP) && !defer && top >= i0 && top < i0 + nbits)
          word |= 1u << (uint32_t)(top - i0);
        cnt += __popc(word);
      }
      s_tr[wid][lane][it] = word;
    }
  }
  __syncwarp();
  uint32_t* brow = a.bitmap + (size_t)r * a.W + wbeg;
  const uint32_t nw = wend - wbeg;
  for (uint32_t it = 0; it < 32; ++it) {
    const uint32_t o = it * 32u + lane;  // word wbeg + o, owned by lane it
    if (o < nw) brow[o] = s_tr[wid][it][lane];
  }
  // per-group counts (group = the 32 words of one lane) for the compaction
  a.task_counts[(size_t)task * 32 + lane] = cnt;
  if (a.fuse_scan && !defer) {  // K2a here: exclusive scan over the 32 groups
    uint64_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    a.task_off[(size_t)task * 32 + lane] = x - cnt;
    if (lane == 31) a.counts[r] = x;
  }
}

// K1n: the noisy router's verdicts over the truth bitmap K1 wrote (router.cpp:
// 50-57): key = mix({seed, 0xA3, id, hash_config(c)}) >> 11
// = absorb(P, hc[c]) >> 11 with hash_config tabulated per space.  One block
// per warp-task, one warp per 4 rows of 32 words; lane j is bit j, so a
// word's 32 table entries are one coalesced 256-byte load and its new
// verdicts are ballots.  Only words holding a bit the noise can change are
// visited, four at a time so their table loads are in flight together.
// Rewrites the changed words and the per-group counts; forces the top
// configuration in (AG_FORCE_TOP).  A separate kernel so the hashing work,
// which varies with each request's truth density, is spread over small
// units instead of whole-request tasks.
constexpr int kNoiseRows = 32 / kWarpsPerBlock;

__global__ void __launch_bounds__(kThreads) k_route_noise(ScoreArgs a) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t task = blockIdx.x;
  const uint32_t r = a.C == 1 ? task : (uint32_t)__umul64hi(task, a.div_c);
  const uint32_t c = task - r * a.C;
  const uint64_t P = absorb(absorb(absorb(kMixIV, a.rt.noise_seed), kRouterSalt), __ldg(a.t.request_ids + r));
  // absorb(P, w) = splitmix(P ^ (w + Pc)) (rng.h:46-49)
  const uint64_t Pc = kGamma + (P << 6) + (P >> 2);
  const bool use_fn = a.rt.t_fn > 0, use_fp = a.rt.t_fp > 0;
  const uint32_t keep_fn = use_fn ? 0xffffffffu : 0u, keep_fp = use_fp ? 0xffffffffu : 0u;
  const uint64_t top = a.sp.size - 1;
  const uint32_t wbeg = c * kTaskWords, wend = min(a.W, wbeg + kTaskWords);
  uint32_t* brow = a.bitmap + (size_t)r * a.W;
  for (int L = wid * kNoiseRows; L < (wid + 1) * kNoiseRows; ++L) {
    const uint32_t wg = wbeg + 32u * (uint32_t)L;  // first word of the row
    if (wg >= wend) break;
    const uint32_t w = wg + lane;                    // lane t: word wg + t
    const uint64_t ib = a.begin + (uint64_t)wg * 32;
    const uint64_t i0 = ib + 32ull * lane;
    const uint32_t valid = (w >= wend || i0 >= a.end) ? 0u
                         : (a.end - i0 >= 32 ? 0xffffffffu : ((1u << (uint32_t)(a.end - i0)) - 1u));
    const uint32_t truth = valid ? brow[w] : 0u;
    uint32_t word = truth;
    uint32_t nz = __ballot_sync(0xffffffffu, (((truth & keep_fn) | (~truth & keep_fp)) & valid) != 0u);
    const uint64_t* hrow = a.hc + ib + lane;  // + 32 t: word t's entries
    // every word of the row full and inside [begin, end): unguarded loads
    const bool rfull = wg + 32 <= wend && ib + 1024 <= a.end;
    auto verdicts = [&](const uint32_t (&t)[4], const uint64_t (&hv)[4], int nb) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (u >= nb) break;  // uniform
        const uint64_t key = splitmix_step(P ^ (hv[u] + Pc)) >> 11;
        const uint32_t tr = __shfl_sync(0xffffffffu, truth, (int)t[u]);
        uint32_t v = tr;
        if (use_fn) v &= __ballot_sync(0xffffffffu, key >= a.rt.t_fn);
        if (use_fp) v |= ~tr & __ballot_sync(0xffffffffu, key < a.rt.t_fp);
        if ((uint32_t)lane == t[u]) word = v & valid;
      }
    };
    while (nz) {
      uint32_t t[4];
      uint64_t hv[4];
      const int nb = min(4, __popc(nz));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        t[u] = nz ? (uint32_t)(__ffs(nz) - 1) : 0u;
        nz &= nz - 1;
      }
      if (rfull && nb == 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) hv[u] = __ldg(hrow + 32 * t[u]);
        verdicts(t, hv, 4);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t ci = ib + 32ull * t[u] + lane;
          hv[u] = (u < nb && ci < a.end) ? __ldg(a.hc + ci) : 0ull;
        }
        verdicts(t, hv, nb);
      }
    }
    if ((a.flags & AG_FORCE_TOP) && valid && top >= i0 && top < i0 + 32) word |= 1u << (uint32_t)(top - i0);
    if (word != truth) brow[w] = word;
    const uint32_t cnt = __reduce_add_sync(0xffffffffu, (uint32_t)__popc(word));
    if (lane == 0) a.task_counts[(size_t)task * 32 + L] = cnt;
  }
  if (a.fuse_scan) {  // K2a here: exclusive scan over the task's 32 groups
    __syncthreads();
    if (wid == 0) {
      const uint32_t v = a.task_counts[(size_t)task * 32 + lane];
      uint64_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      a.task_off[(size_t)task * 32 + lane] = x - v;
      if (lane == 31) a.counts[r] = x;
    }
  }
}

// K2a: one warp per request: exclusive scan of its group counts (32 per
// warp-task) -> group offsets relative to the request, counts[r] = total.
__global__ void __launch_bounds__(kThreads)
    k_chunk_scan(const uint32_t* __restrict__ task_counts, uint64_t* __restrict__ task_off,
                 uint64_t* __restrict__ counts, uint32_t C, int R) {
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (r >= R) return;
  const uint32_t* in = task_counts + (size_t)r * C;
  uint64_t* out = task_off + (size_t)r * C;
  uint64_t carry = 0;
  for (uint32_t base = 0; base < C; base += 32) {
    const uint32_t i = base + lane;
    const uint64_t v = i < C ? in[i] : 0u;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (i < C) out[i] = carry + (x - v);
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) counts[r] = carry;
}

// K2a for deep spaces (more than 4096 groups per request): each request's
// group counts are split into kScanSlices slices, so R * kScanSlices blocks
// share the work.  Pass 1 sums every slice (coalesced); pass 2 scans each
// slice from its base (the sum of the earlier slices of its request) in
// tiles of 8 * 1024 counts staged through shared memory, and the last slice
// writes the request total.
constexpr int kScanSlices = 16;
constexpr int kScanPer = 8;  // counts per thread per tile

__global__ void __launch_bounds__(1024)
    k_chunk_partial(const uint32_t* __restrict__ task_counts, uint64_t* __restrict__ part, uint32_t C) {
  __shared__ uint64_t warp_sums[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t r = blockIdx.y, p = blockIdx.x;
  const uint32_t slice = (C + kScanSlices - 1) / kScanSlices;
  const uint32_t lo = min(C, p * slice), hi = min(C, lo + slice);
  const uint32_t* in = task_counts + (size_t)r * C;
  uint64_t x = 0;
  for (uint32_t i = lo + threadIdx.x; i < hi; i += 1024) x += __ldg(in + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (lane == 0) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint64_t v = warp_sums[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) part[(size_t)r * kScanSlices + p] = v;
  }
}

__global__ void __launch_bounds__(1024)
    k_chunk_scan_slices(const uint32_t* __restrict__ task_counts, const uint64_t* __restrict__ part,
                        uint64_t* __restrict__ task_off, uint64_t* __restrict__ counts, uint32_t C) {
  __shared__ uint32_t s_in[kScanPer * 1024];
  __shared__ uint64_t warp_sums[32];
  __shared__ uint64_t s_base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t r = blockIdx.y, p = blockIdx.x;
  const uint32_t slice = (C + kScanSlices - 1) / kScanSlices;
  const uint32_t lo = min(C, p * slice), hi = min(C, lo + slice);
  const uint32_t* in = task_counts + (size_t)r * C;
  uint64_t* out = task_off + (size_t)r * C;
  if (wid == 0) {
    const uint64_t v = lane < (int)p ? part[(size_t)r * kScanSlices + lane] : 0ull;
    uint64_t z = v;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    if (lane == 0) s_base = z;
    if (p == kScanSlices - 1 && lane == 0) {
      uint64_t tot = 0;
      for (int q = 0; q < kScanSlices; ++q) tot += part[(size_t)r * kScanSlices + q];
      counts[r] = tot;
    }
  }
  __syncthreads();
  uint64_t carry = s_base;
  for (uint32_t t0 = lo; t0 < hi; t0 += kScanPer * 1024) {
    const uint32_t n = min(hi - t0, (uint32_t)(kScanPer * 1024));
#pragma unroll
    for (int u = 0; u < kScanPer; ++u) {
      const uint32_t i = u * 1024 + threadIdx.x;
      s_in[i] = i < n ? __ldg(in + t0 + i) : 0u;
    }
    __syncthreads();
    uint32_t v[kScanPer];
    uint64_t local = 0;
#pragma unroll
    for (int u = 0; u < kScanPer; ++u) {
      v[u] = s_in[threadIdx.x * kScanPer + u];
      local += v[u];
    }
    uint64_t x = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const uint64_t w = warp_sums[lane];
      uint64_t z = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      warp_sums[lane] = z - w;  // exclusive warp prefix
    }
    __syncthreads();
    uint64_t run = carry + warp_sums[wid] + x - local;
    const uint32_t b = threadIdx.x * kScanPer;
#pragma unroll
    for (int u = 0; u < kScanPer; ++u) {
      if (b + u < n) out[t0 + b + u] = run;
      run += v[u];
    }
    // the tile total, for the next tile's carry
    __syncthreads();  // every thread has read its warp prefix
    if (threadIdx.x == 1023) warp_sums[0] = run;  // run after the last element
    __syncthreads();
    carry = warp_sums[0];
    __syncthreads();
  }
}

// K2b: exclusive scan over requests -> offsets[R+1], overflow flag.  One
// block, tiles of PER x 1024 counts (PER picked so a batch is one tile up to
// 24k requests: every load of the batch is in flight at once, then one
// scan): loaded and stored coalesced through shared memory (a single SM's L1
// is the limit: per-thread contiguous runs would cost one sector request per
// element), each thread scanning PER contiguous counts of the tile; the tile
// total carries to the next tile.
template <int kReqPer>
__global__ void __launch_bounds__(1024)
    k_request_scan(const uint64_t* __restrict__ counts, uint64_t* __restrict__ offsets, int R,
                   uint64_t capacity, uint32_t* __restrict__ overflow) {
  extern __shared__ uint64_t s_t[];  // [kReqPer * 1024]
  __shared__ uint64_t warp_sums[32];
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's counts
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t carry = 0;
  for (int t0 = 0; t0 < R; t0 += kReqPer * 1024) {
    const int n = min(R - t0, kReqPer * 1024);
#pragma unroll
    for (int u = 0; u < kReqPer; ++u) {
      const int i = u * 1024 + threadIdx.x;
      s_t[i] = i < n ? __ldg(counts + t0 + i) : 0ull;
    }
    __syncthreads();
    uint64_t local = 0;
#pragma unroll
    for (int u = 0; u < kReqPer; ++u) local += s_t[threadIdx.x * kReqPer + u];
    uint64_t x = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const uint64_t w = warp_sums[lane];
      uint64_t z = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      warp_sums[lane] = z - w;  // exclusive warp prefix
    }
    __syncthreads();
    uint64_t run = carry + warp_sums[wid] + x - local;
#pragma unroll
    for (int u = 0; u < kReqPer; ++u) {
      const uint64_t c = s_t[threadIdx.x * kReqPer + u];
      s_t[threadIdx.x * kReqPer + u] = run;
      run += c;
    }
    __syncthreads();  // tile offsets staged; every warp prefix read
#pragma unroll
    for (int u = 0; u < kReqPer; ++u) {
      const int i = u * 1024 + threadIdx.x;
      if (i < n) offsets[t0 + i] = s_t[i];
    }
    if (threadIdx.x == 1023) warp_sums[0] = run;  // the running total after this tile
    __syncthreads();
    carry = warp_sums[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    offsets[R] = carry;
    if (overflow) *overflow = carry > capacity ? 1u : 0u;
  }
}

// Programmatic dependent launch: the kernel may begin while the previous
// kernel on the stream still runs; it waits (griddepcontrol.wait) for that
// grid's completion and memory before touching its outputs.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
}

cudaError_t launch_request_scan(ag_ctx* ctx, cudaStream_t s, const uint64_t* counts, uint64_t* offsets, int R,
                                uint64_t capacity, uint32_t* overflow) {
  bool& attr = ctx->scan_attr;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_request_scan<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 1024 * 8);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_request_scan<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 1024 * 8);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  if (R <= 4 * 1024)
    return launch_pdl(k_request_scan<4>, 1, 1024, 4 * 1024 * 8, s, counts, offsets, R, capacity, overflow);
  if (R <= 12 * 1024)
    return launch_pdl(k_request_scan<12>, 1, 1024, 12 * 1024 * 8, s, counts, offsets, R, capacity, overflow);
  return launch_pdl(k_request_scan<24>, 1, 1024, 24 * 1024 * 8, s, counts, offsets, R, capacity, overflow);
}

// K3: stream compaction of the verdict bitmap into canonical-order indices.
// Work unit = unit_groups_for(W) groups of 32 words (each group's output offset is
// known from K2a); persistent warps stride over units.  Per iteration the warp
// loads 32 words (coalesced, software-pipelined) and scans their popcounts;
// the members are staged bit-parallel in shared memory -- for word w lane j
// stores member (w, j) at prefix(w) + popc(word_w & lanemask_lt), a
// conflict-free contiguous run, with words / prefixes read four at a time by
// broadcast 16-byte loads -- aligned to the output's 16-byte phase, and every
// full 16-byte vector is written back at once; the <= 3 trailing members carry
// over to the next iteration, so global stores are almost all full vectors.
constexpr int kStage = 32 * 32 + 8;  // one iteration's members + carry + pad
// groups per unit: 4 for rows of up to 2^16 words (config 2: finer units
// balance the per-request density spread), 16 for deep rows (config 4: the
// per-unit start amortised over more words); AG_UNIT_GROUPS forces one
// (scripts/compact_sweep*.sh, profiles/r02w_compact_unit_sweep.txt)
#ifndef AG_UNIT_GROUPS
#define AG_UNIT_GROUPS 0
#endif
constexpr uint32_t unit_groups_for(uint32_t W) {  // 2, 4, 8 or 16 (instantiated)
  return AG_UNIT_GROUPS > 0 ? (uint32_t)AG_UNIT_GROUPS : (W <= (1u << 16) ? 4u : 16u);
}

template <uint32_t ug>
__global__ void __launch_bounds__(kThreads)
    k_route_compact(const uint32_t* __restrict__ bitmap, const uint64_t* __restrict__ group_off,
                    const uint64_t* __restrict__ offsets, uint64_t begin, uint32_t W, uint32_t C,
                    uint32_t units_per_req, uint64_t div_u, int R, uint32_t* __restrict__ indices,
                    uint64_t capacity) {
  __shared__ __align__(16) uint32_t s_stage[kWarpsPerBlock][kStage];
  __shared__ __align__(16) uint32_t s_word[kWarpsPerBlock][32];
  __shared__ __align__(16) uint32_t s_pre[kWarpsPerBlock][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t lt = (1u << lane) - 1u, bit = 1u << lane;
  uint32_t* st = s_stage[wid];
  asm volatile("griddepcontrol.wait;" ::: "memory");  // K1's bitmap, K2's offsets
  const uint64_t units = (uint64_t)R * units_per_req;
  const uint32_t nwarps = gridDim.x * kWarpsPerBlock;
  // a unit's request and its output position; the next unit's are loaded
  // while the current one is processed (two dependent global loads)
  auto unit_of = [&](uint64_t unit, uint32_t& r, uint32_t& g0) {
    r = units_per_req == 1 ? (uint32_t)unit : (uint32_t)__umul64hi(unit, div_u);
    g0 = ((uint32_t)unit - r * units_per_req) * ug;  // first group (32 words each)
  };
  uint64_t unit = (uint64_t)blockIdx.x * kWarpsPerBlock + wid;
  uint64_t gs_next = 0;
  if (unit < units) {
    uint32_t r, g0;
    unit_of(unit, r, g0);
    gs_next = __ldg(offsets + r) + __ldg(group_off + (size_t)r * C * 32 + g0);
  }
  for (; unit < units; unit += nwarps) {
    uint32_t r, g0;
    unit_of(unit, r, g0);
    const uint32_t wbeg = g0 * 32;
    const uint32_t wend = min(W, wbeg + 32 * ug);
    // global output position of the unit's first member
    const uint64_t gs = gs_next;
    if (unit + nwarps < units) {
      uint32_t r2, g2;
      unit_of(unit + nwarps, r2, g2);
      gs_next = __ldg(offsets + r2) + __ldg(group_off + (size_t)r2 * C * 32 + g2);
    }
    const uint32_t* brow = bitmap + (size_t)r * W;
    const uint32_t phase0 = (uint32_t)(reinterpret_cast<uintptr_t>(indices + gs) >> 2) & 3u;
    uint32_t* gal = indices + (gs - phase0);  // 16-byte aligned output cursor (stage[0])
    uint64_t gpos = gs - phase0;              // its global index
    uint32_t fill = phase0;  // stage[0, fill): carried members (or, at first, not ours)
    uint32_t skip = phase0;  // leading stage entries that are not ours (first vector only)
    // bitmap words two iterations ahead (empty iterations are short)
    uint32_t next = wbeg + lane < wend ? __ldg(brow + wbeg + lane) : 0u;
    uint32_t next2 = wbeg + 32 + lane < wend ? __ldg(brow + wbeg + 32 + lane) : 0u;
    uint32_t carry = 0;  // lanes < fill: the members carried into the next vector
    for (uint32_t wb = wbeg; wb < wend; wb += 32) {
      const uint32_t word = next;
      next = next2;
      const uint32_t wn = wb + 64 + lane;
      next2 = wn < wend ? __ldg(brow + wn) : 0u;
      const uint32_t pc = __popc(word);
      uint32_t x = pc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, x, 31);
      if (total == 0) continue;
      // the stage is rewritten: the previous bulk store must have read it
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      if (lane < fill) st[lane] = carry;
      s_word[wid][lane] = word;
      s_pre[wid][lane] = x - pc + fill;
      __syncwarp();
      const uint32_t vl = (uint32_t)(begin + (uint64_t)wb * 32) + (uint32_t)lane;
#pragma unroll
      for (int w4 = 0; w4 < 32; w4 += 4) {
        const uint4 ww = *reinterpret_cast<const uint4*>(&s_word[wid][w4]);
        const uint4 pp = *reinterpret_cast<const uint4*>(&s_pre[wid][w4]);
        if (ww.x & bit) st[pp.x + __popc(ww.x & lt)] = vl + 32u * (w4 + 0);
        if (ww.y & bit) st[pp.y + __popc(ww.y & lt)] = vl + 32u * (w4 + 1);
        if (ww.z & bit) st[pp.z + __popc(ww.z & lt)] = vl + 32u * (w4 + 2);
        if (ww.w & bit) st[pp.w + __popc(ww.w & lt)] = vl + 32u * (w4 + 3);
      }
      // the staged members become visible to the bulk-copy (async) proxy
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      // full vectors now, as one bulk store (TMA engine: shared -> global,
      // 16-byte aligned on both sides); the partial last vector carries over
      const uint32_t end = fill + total;
      const uint32_t nfull = end >> 2;
      const bool in_cap = gpos + 4ull * nfull <= capacity;
      const uint32_t v0 = skip ? 1u : 0u;  // a first vector holding entries not ours goes per lane
      if (in_cap && nfull > v0) {
        if (lane == 0) {
          const uint32_t saddr = (uint32_t)__cvta_generic_to_shared(st + 4 * v0);
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                       "cp.async.bulk.commit_group;" ::"l"(gal + 4 * v0), "r"(saddr), "r"(16u * (nfull - v0))
                       : "memory");
        }
        if (v0 && lane < 4 && lane >= skip) gal[lane] = st[lane];
      } else {
        for (uint32_t e = lane; e < 4 * nfull; e += 32)
          if (e >= skip && gpos + e < capacity) gal[e] = st[e];
      }
      const uint32_t tail = end & 3u;
      carry = lane < tail ? st[4 * nfull + lane] : 0u;
      if (nfull) skip = 0;
      fill = tail;
      gal += 4 * nfull;
      gpos += 4ull * nfull;
    }
    // the last partial vector
    if (lane >= skip && lane < fill && gpos + lane < capacity) gal[lane] = carry;
    __syncwarp();
  }
  // every bulk store complete before the warp's stage goes away
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __syncwarp();
}

template <int NT>
void launch_score(dim3 g, cudaStream_t s, const ScoreArgs& a) {
  k_route_score<NT><<<g, kThreads, 0, s>>>(a);
}

typedef void (*score_fn)(dim3, cudaStream_t, const ScoreArgs&);

score_fn pick_score(int n) {
  switch (n) {
    case 1: return launch_score<1>;
    case 2: return launch_score<2>;
    case 3: return launch_score<3>;
    case 4: return launch_score<4>;
    case 5: return launch_score<5>;
    case 6: return launch_score<6>;
    case 7: return launch_score<7>;
    case 8: return launch_score<8>;
    case 9: return launch_score<9>;
    case 10: return launch_score<10>;
    case 11: return launch_score<11>;
    case 12: return launch_score<12>;
    default: return launch_score<0>;
  }
}

// ceil(2^64 / d) for exact u32 division via __umul64hi; d <= 1 is handled
// by the callers (C == 1 means task == request)
inline uint64_t magic_div(uint32_t d) { return d > 1 ? (~0ULL) / (uint64_t)d + 1 : 0; }

// colmask[l0][c] = positions j in 0..31 with (l0 + j) mod M >= c
// hash_config(c) (router.cpp:22-28) for every canonical index: the noisy
// router's per-configuration state does not depend on the request, so it is
// tabulated once per space (spaces up to kHashTableMax configurations).
constexpr uint64_t kHashTableMax = 1ull << 24;

__global__ void k_hash_table(SpaceDev sp, uint64_t* __restrict__ hc) {
  const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= sp.size) return;
  uint32_t d[kMaxAgents];
  uint32_t x = (uint32_t)c;
  for (int a = sp.n - 1; a >= 0; --a) {
    const uint32_t q = divm(x, sp.div_m);
    d[a] = x - q * (uint32_t)sp.m;
    x = q;
  }
  uint64_t h = kHashIV;
  for (int a = 0; a < sp.n; ++a) h = absorb(absorb(kMixIV, h), d[a]);  // mix({h, m})
  hc[c] = h;
}

const uint64_t* ensure_hash_table(ag_ctx* ctx) {
  const ag_space* sp = ctx->space;
  if (sp->size > kHashTableMax) return nullptr;
  if (!ctx->hc_ready) {
    if (ctx->hc.ensure(8 * sp->size + 8)) return nullptr;
    const unsigned blocks = (unsigned)((sp->size + 255) / 256);
    k_hash_table<<<blocks, 256, 0, ctx->stream>>>(sp->dev(), (uint64_t*)ctx->hc.p);
    if (cudaGetLastError() != cudaSuccess) return nullptr;
    ctx->hc_ready = true;
  }
  return (const uint64_t*)ctx->hc.p;
}

int ensure_colmask(ag_ctx* ctx) {
  const int m = ctx->space->m;
  if (ctx->colmask.bytes >= 32 * 32 * 4 && ctx->colmask_m == m) return AG_OK;
  std::vector<uint32_t> h(32 * 32, 0);
  for (int l0 = 0; l0 < m && l0 < 32; ++l0)
    for (int c = 0; c < m && c < 32; ++c) {
      uint32_t bits = 0;
      for (int j = 0; j < 32; ++j)
        if ((l0 + j) % m >= c) bits |= 1u << j;
      h[l0 * 32 + c] = bits;
    }
  int rc = ctx->colmask.ensure(h.size() * 4);
  if (rc) return rc;
  AG_CUDA(cudaMemcpy(ctx->colmask.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
  ctx->colmask_m = m;
  return AG_OK;
}

}  // namespace

int make_router(const ag_router* r, RouterDev* out) {
  if (!r) return fail(AG_ERR_VALIDATION, "router is null");
  RouterDev d{};
  d.kind = r->kind;
  d.noise_seed = r->noise_seed;
  if (r->eval_latency < 0) return fail(AG_ERR_VALIDATION, "router eval latency < 0");
  if (r->kind == AG_ROUTER_NOISY) {
    // NoisyRouter ctor check (router.cpp:41-48); NaN passes it there, and a
    // NaN rate makes the corresponding comparison always false.
    if (r->fp < 0 || r->fp > 1 || r->fn < 0 || r->fn > 1)
      return fail(AG_ERR_VALIDATION, "router error rates outside [0, 1]");
    d.t_fn = std::isnan(r->fn) ? ~0ULL : (uint64_t)std::ceil(r->fn * 0x1.0p53);
    d.t_fp = std::isnan(r->fp) ? 0ULL : (uint64_t)std::ceil(r->fp * 0x1.0p53);
  } else if (r->kind != AG_ROUTER_ORACLE) {
    return fail(AG_ERR_VALIDATION, "unknown router kind");
  }
  *out = d;
  return AG_OK;
}

// K3 launch: persistent warps over units of unit_groups_for(W) groups, the grid
// sized to the device's resident capacity for this kernel.
int launch_compact(ag_ctx* ctx, int R, uint32_t W, uint32_t C, uint64_t begin, const uint32_t* bitmap,
                   const uint64_t* offsets, uint32_t* indices, uint64_t capacity) {
  int& resident = ctx->compact_resident;  // blocks per device (SMs x blocks per SM)
  if (!resident) {
    int sms = 0, per_sm = 0;
    AG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    AG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_route_compact<4>, kThreads, 0));
    resident = std::max(1, sms * per_sm);
  }
  const uint32_t ngroups = (W + 31) / 32;
  const uint32_t ug = unit_groups_for(W);
  const uint32_t upr = (ngroups + ug - 1) / ug;
  const uint64_t units = (uint64_t)R * upr;
  if (units >= (1ULL << 32)) return fail(AG_ERR_VALIDATION, "batch too large for one launch");
  const uint64_t want = (units + kWarpsPerBlock - 1) / kWarpsPerBlock;
  const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)resident));
  Launch L(ctx, K_ROUTE_COMPACT);
  auto* kern = ug == 16 ? k_route_compact<16> : ug == 8 ? k_route_compact<8> : ug == 2 ? k_route_compact<2>
                                                                               : k_route_compact<4>;
  AG_CUDA(launch_pdl(kern, blocks, kThreads, 0, ctx->stream, bitmap, (const uint64_t*)ctx->chunk_off.p, offsets,
                     begin, W, C, upr, magic_div(upr), R, indices, capacity));
  return AG_OK;
}

int route_enumerate(ag_ctx* ctx, const ag_truth* t, const ag_router* r, uint64_t begin,
                    uint64_t end, uint32_t flags, const ag_route_out* out) {
  const ag_space* sp = ctx->space;
  if (!t || !out) return fail(AG_ERR_VALIDATION, "null truth/out");
  if (!sp->gpu_ok) return fail(AG_ERR_VALIDATION, "GPU path needs M^N <= 2^32 and N <= 32");
  if (begin > end || end > sp->size) return fail(AG_ERR_VALIDATION, "configuration index out of range");
  if (t->n_requests < 0) return fail(AG_ERR_VALIDATION, "negative request count");
  RouterDev rt;
  int rc = make_router(r, &rt);
  if (rc) return rc;
  const int R = t->n_requests;
  cudaStream_t s = ctx->stream;
  if (R == 0) {
    if (out->offsets) AG_CUDA(cudaMemsetAsync(out->offsets, 0, 8, s));
    if (out->overflow) AG_CUDA(cudaMemsetAsync(out->overflow, 0, 4, s));
    return AG_OK;
  }
  if (!out->counts) return fail(AG_ERR_VALIDATION, "counts output is required");
  const uint64_t range = end - begin;
  const uint32_t W = (uint32_t)((range + 31) / 32);
  const uint32_t C = (W + kTaskWords - 1) / kTaskWords;
  const uint64_t ntasks = (uint64_t)R * C;
  if (ntasks >= (1ULL << 31)) return fail(AG_ERR_VALIDATION, "batch too large for one launch");

  if ((rc = ctx->chunk_counts.ensure(ntasks * 32 * 4))) return rc;
  if ((rc = ctx->chunk_off.ensure(ntasks * 32 * 8))) return rc;
  if ((rc = ensure_colmask(ctx))) return rc;
  uint32_t* bitmap = out->bitmap;
  if (!bitmap) {
    if ((rc = ctx->bitmap.ensure((size_t)R * W * 4 + 4))) return rc;
    bitmap = (uint32_t*)ctx->bitmap.p;
  }
  uint64_t* offsets = out->offsets;
  if (!offsets) {
    if ((rc = ctx->offsets.ensure(((size_t)R + 1) * 8))) return rc;
    offsets = (uint64_t*)ctx->offsets.p;
  }
  ScoreArgs a;
  a.sp = sp->dev();
  a.t = TruthDev{R, t->request_ids, t->seed_ptr, t->seeds, t->removed_ptr, t->removed};
  a.rt = rt;
  a.begin = begin;
  a.end = end;
  a.W = W;
  a.C = C;
  a.div_c = magic_div(C);
  a.R = R;
  a.flags = flags;
  a.H = 0;
  for (int b = 0; b < sp->n - 2 && b < 8; ++b) a.H |= 0x80ull << (8 * b);
  a.path2d = (sp->n >= 2 && sp->n - 2 <= 8 && sp->m <= 32) ? 1 : 0;
  {
    // phase-pattern path: blocks of >= 32 indices, <= kPatMax phases
    const uint32_t Bq = (uint32_t)sp->m * (uint32_t)sp->m;
    uint32_t g = 1;
    while (g < 32 && Bq % (2 * g) == 0) g *= 2;
    a.pat_P = (int)(Bq / g);
    a.pat_lg = (a.path2d && Bq >= 32 && a.pat_P <= kPatMax) ? __builtin_ctz(g) : -1;
  }
  a.colmask = (const uint32_t*)ctx->colmask.p;
  a.hc = rt.kind == AG_ROUTER_NOISY ? ensure_hash_table(ctx) : nullptr;
  a.bitmap = bitmap;
  a.task_counts = (uint32_t*)ctx->chunk_counts.p;
  a.fuse_scan = C == 1 ? 1 : 0;
  a.task_off = (uint64_t*)ctx->chunk_off.p;
  a.counts = out->counts;
  const dim3 grid((unsigned)((ntasks + kWarpsPerBlock - 1) / kWarpsPerBlock));
  if (range > 0) {
    {
      Launch L(ctx, K_ROUTE_SCORE);
      pick_score(sp->n)(grid, s, a);
    }
    if (a.hc) {  // noisy router: verdicts over the truth bitmap
      Launch L(ctx, K_ROUTE_NOISE);
      k_route_noise<<<(unsigned)ntasks, kThreads, 0, s>>>(a);
    }
  } else {
    AG_CUDA(cudaMemsetAsync(out->counts, 0, (size_t)R * 8, s));
    Launch L(ctx, K_REQUEST_SCAN);
    AG_CUDA(launch_request_scan(ctx, s, out->counts, offsets, R, out->indices ? out->capacity : ~0ULL, out->overflow));
    AG_CUDA(cudaGetLastError());
    return AG_OK;
  }
  return finish_enumerate(ctx, R, W, C, begin, bitmap, offsets, out, a.fuse_scan != 0);
}

// K2 scans + K3 compaction of a verdict bitmap [R][W] whose per-group counts
// ([R][C*32], 32-word groups) are in ctx->chunk_counts: shared by the oracle /
// noisy scoring kernel and the learned router (ag_linear.cu).
int finish_enumerate(ag_ctx* ctx, int R, uint32_t W, uint32_t C, uint64_t begin, uint32_t* bitmap,
                     uint64_t* offsets, const ag_route_out* out, bool scanned) {
  cudaStream_t s = ctx->stream;
  if (scanned) {
    // group offsets and counts already written by the scoring kernel
  } else if (C * 32 <= 4096) {
    Launch L(ctx, K_CHUNK_SCAN);
    k_chunk_scan<<<(R + kWarpsPerBlock - 1) / kWarpsPerBlock, kThreads, 0, s>>>(
        (const uint32_t*)ctx->chunk_counts.p, (uint64_t*)ctx->chunk_off.p, out->counts, C * 32, R);
  } else {
    int rc = ctx->chunk_part.ensure((size_t)R * kScanSlices * 8);
    if (rc) return rc;
    const dim3 g(kScanSlices, R);
    {
      Launch L(ctx, K_CHUNK_SCAN);
      k_chunk_partial<<<g, 1024, 0, s>>>((const uint32_t*)ctx->chunk_counts.p,
                                         (uint64_t*)ctx->chunk_part.p, C * 32);
    }
    Launch L(ctx, K_CHUNK_SCAN);
    k_chunk_scan_slices<<<g, 1024, 0, s>>>((const uint32_t*)ctx->chunk_counts.p,
                                           (const uint64_t*)ctx->chunk_part.p,
                                           (uint64_t*)ctx->chunk_off.p, out->counts, C * 32);
  }
  {
    Launch L(ctx, K_REQUEST_SCAN);
    AG_CUDA(launch_request_scan(ctx, s, out->counts, offsets, R, out->indices ? out->capacity : ~0ULL, out->overflow));
  }
  if (out->indices) {
    const int rc = launch_compact(ctx, R, W, C, begin, bitmap, offsets, out->indices, out->capacity);
    if (rc) return rc;
  }
  AG_CUDA(cudaGetLastError());
  return AG_OK;
}

// Compaction pass alone, reusing the group offsets of the preceding
// route_enumerate on this context (the host path's second phase).
int route_compact(ag_ctx* ctx, int R, uint64_t begin, uint64_t end, const uint32_t* bitmap,
                  const uint64_t* offsets, uint32_t* indices, uint64_t capacity) {
  const uint64_t range = end - begin;
  if (R == 0 || range == 0) return AG_OK;
  const uint32_t W = (uint32_t)((range + 31) / 32);
  const uint32_t C = (W + kTaskWords - 1) / kTaskWords;
  return launch_compact(ctx, R, W, C, begin, bitmap, offsets, indices, capacity);
}

}  // namespace agb

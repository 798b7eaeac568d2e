// H2 boundary input, native: bit-exact port of the reference's stratified
// draws (strata.py:113-161) and seed derivation (seeding.py:7-21), host C++.
//
// The reference draws with numpy's Generator (PCG64 seeded by SeedSequence)
// and `rng.choice(len(pool), take, replace=False)` (strata.py:147); the picked
// indices are then swap-popped in descending order (:148-152) and a dry
// stratum borrows from the nonempty stratum with the closest boundary
// (:131-140, :155-161).  Everything here restates numpy 2.x's published
// algorithms (numpy/random: bit_generator.pyx SeedSequence, pcg64.c,
// distributions.c random_bounded_uint64 / Lemire, _generator.pyx choice:
// tail shuffle or Floyd + shuffle) and is differential-tested against the
// installed numpy (tests/test_draws.py); it replaces a Python loop running
// at 0.06-0.27 M keys/s.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "b2ddp.h"
#include "rng.h"

namespace b2 {
void set_error(const char* fmt, ...);
}

namespace {

using namespace b2::rng;

struct Pcg64H : Pcg64 {  // host extras: numpy's shuffle and choice(replace=False)
  using Pcg64::Pcg64;
  void shuffle_int(int64_t n, int64_t first, int64_t* data) {  // _shuffle_int
    for (int64_t i = n - 1; i >= first; --i) {
      const int64_t j = (int64_t)bounded((uint64_t)i);
      const int64_t t = data[j];
      data[j] = data[i];
      data[i] = t;
    }
  }
  // Generator.choice(pop, size, replace=False, shuffle=True) -> size indices
  void choice(int64_t pop, int64_t size, std::vector<int64_t>& out, std::vector<int64_t>& scratch,
              std::vector<uint64_t>& set) {
    out.resize(size);
    if (size == 0) return;
    // branch rule of numpy 2.x (verified against the installed numpy over a
    // grid of (pop, size), tests/test_draws.py): tail shuffle only for large
    // populations with a large sample, Floyd otherwise
    if (pop > 10000 && size > pop / 50) {  // tail shuffle
      scratch.resize(pop);
      for (int64_t i = 0; i < pop; ++i) scratch[i] = i;
      shuffle_int(pop, pop - size > 1 ? pop - size : 1, scratch.data());
      memcpy(out.data(), scratch.data() + (pop - size), sizeof(int64_t) * size);
    } else {  // Floyd's algorithm with an open-addressing set, then shuffle
      uint64_t mask = (uint64_t)(1.2 * (double)size);
      mask |= mask >> 1;
      mask |= mask >> 2;
      mask |= mask >> 4;
      mask |= mask >> 8;
      mask |= mask >> 16;
      mask |= mask >> 32;
      set.assign(mask + 1, ~0ull);
      for (int64_t j = pop - size; j < pop; ++j) {
        const uint64_t val = bounded((uint64_t)j);
        uint64_t loc = val & mask;
        while (set[loc] != ~0ull && set[loc] != val) loc = (loc + 1) & mask;
        if (set[loc] == ~0ull) {
          set[loc] = val;
          out[j - pop + size] = (int64_t)val;
        } else {
          loc = (uint64_t)j & mask;
          while (set[loc] != ~0ull) loc = (loc + 1) & mask;
          set[loc] = (uint64_t)j;
          out[j - pop + size] = j;
        }
      }
      shuffle_int(size, 1, out.data());
    }
  }
};

}  // namespace

struct b2_draw_state {
  std::vector<std::vector<int64_t>> pools;  // per-stratum ids, mutated by draws (strata.py:26-28)
  std::vector<int64_t> bounds;
  std::vector<int64_t> picked, scratch;
  std::vector<uint64_t> set;
};

extern "C" uint64_t b2_derive_seed(uint64_t seed, const uint64_t* key, int nkey) {
  // seeding.py:18-21: SeedSequence(seed, spawn_key=key).generate_state(1, uint64)[0]
  SeedSeq ss(seed, key, nkey);
  uint64_t v;
  ss.generate_u64(&v, 1);
  return v;
}

extern "C" int b2_draws_create(b2_draw_state** out, const int64_t* ids, const int64_t* pool_sizes, int nstrata,
                               const int64_t* bounds) {
  if (!out || !pool_sizes || !bounds || nstrata < 1) {
    b2::set_error("b2_draws_create: bad arguments");
    return B2_ERR_INVALID;
  }
  b2_draw_state* st = new b2_draw_state();
  st->pools.resize(nstrata);
  int64_t o = 0;
  for (int k = 0; k < nstrata; ++k) {
    st->pools[k].assign(ids + o, ids + o + pool_sizes[k]);
    o += pool_sizes[k];
  }
  st->bounds.assign(bounds, bounds + nstrata);
  *out = st;
  return B2_OK;
}

extern "C" int b2_draws_destroy(b2_draw_state* st) {
  delete st;
  return B2_OK;
}

extern "C" int64_t b2_draws_remaining(const b2_draw_state* st, int k) {
  return st && k >= 0 && k < (int)st->pools.size() ? (int64_t)st->pools[k].size() : -1;
}

// One draw_batch (strata.py:113-141): counts[nstrata] -> out[sum(counts)] ids.
// Returns B2_OK, or B2_ERR_INVALID with *err_stratum = k+1 / *err_short on
// global exhaustion (the reference's "stratum k exhausted ..." ValueError).
static int draw_one(b2_draw_state* st, const int64_t* counts, uint64_t seed, int64_t* out, int* err_stratum,
                    int64_t* err_short) {
  Pcg64H rng(seed);
  const int S = (int)st->pools.size();
  int64_t w = 0;
  auto take_from = [&](std::vector<int64_t>& pool, int64_t take) {
    if (take == 0) return;
    rng.choice((int64_t)pool.size(), take, st->picked, st->scratch, st->set);
    std::vector<int64_t>& pk = st->picked;
    // swap-pop in descending index order keeps lower indices valid (:148-152)
    std::sort(pk.begin(), pk.end(), [](int64_t a, int64_t b) { return a > b; });
    for (int64_t i : pk) {
      out[w++] = pool[i];
      pool[i] = pool.back();
      pool.pop_back();
    }
  };
  for (int k = 0; k < S; ++k) {
    const int64_t need = counts[k];
    int64_t take = need < (int64_t)st->pools[k].size() ? need : (int64_t)st->pools[k].size();
    take_from(st->pools[k], take);
    int64_t shortfall = need - take;
    while (shortfall > 0) {
      int best = -1;  // min (|boundary diff|, j) over nonempty j != k (:155-161)
      int64_t bestd = 0;
      for (int j = 0; j < S; ++j) {
        if (j == k || st->pools[j].empty()) continue;
        const int64_t d = st->bounds[j] > st->bounds[k] ? st->bounds[j] - st->bounds[k] : st->bounds[k] - st->bounds[j];
        if (best < 0 || d < bestd) {
          best = j;
          bestd = d;
        }
      }
      if (best < 0) {
        if (err_stratum) *err_stratum = k + 1;
        if (err_short) *err_short = shortfall;
        b2::set_error("stratum %d exhausted and no other stratum can cover the remaining %lld sample(s)", k + 1,
                      (long long)shortfall);
        return B2_ERR_INVALID;
      }
      take = shortfall < (int64_t)st->pools[best].size() ? shortfall : (int64_t)st->pools[best].size();
      take_from(st->pools[best], take);
      shortfall -= take;
    }
  }
  return B2_OK;
}

extern "C" int b2_draw_batch(b2_draw_state* st, const int64_t* counts, uint64_t seed, int64_t* out,
                             int* err_stratum, int64_t* err_short) {
  if (!st || !counts || !out) {
    b2::set_error("b2_draw_batch: bad arguments");
    return B2_ERR_INVALID;
  }
  return draw_one(st, counts, seed, out, err_stratum, err_short);
}

// A run of steps: step t draws with seed derive_seed(base, key..., t) — the
// per-(rank, step) stream the bench and the data loader use.  Returns the
// number of completed steps in *done (stops at exhaustion, which is reported
// like b2_draw_batch).
extern "C" int b2_draw_epoch(b2_draw_state* st, const int64_t* counts, uint64_t base_seed, const uint64_t* key,
                             int nkey, int64_t first_step, int64_t nsteps, int64_t* out, int64_t* done,
                             int* err_stratum, int64_t* err_short) {
  if (!st || !counts || !out || !done || nkey < 0 || nkey > 7) {  // key + step <= 8 words
    b2::set_error("b2_draw_epoch: bad arguments");
    return B2_ERR_INVALID;
  }
  int64_t lb = 0;
  for (size_t k = 0; k < st->pools.size(); ++k) lb += counts[k];
  uint64_t kk[8];
  for (int i = 0; i < nkey; ++i) kk[i] = key[i];
  *done = 0;
  for (int64_t t = 0; t < nsteps; ++t) {
    kk[nkey] = (uint64_t)(first_step + t);
    const uint64_t seed = b2_derive_seed(base_seed, kk, nkey + 1);
    const int rc = draw_one(st, counts, seed, out + t * lb, err_stratum, err_short);
    if (rc != B2_OK) return rc;
    *done = t + 1;
  }
  return B2_OK;
}

// ---------------------------------------------------------------- Monte-Carlo trials
// mcsim.py (the balance experiment's per-trial draws): trial t uses
// derive_rng(seed, t) = default_rng(SeedSequence(seed, spawn_key=(t,)))
// (seeding.py:8-16).  For each stratum k with counts[k] > 0, in order,
// need = counts[k] * G lengths are drawn as lens_k[choice(|pool_k|, need,
// replace=False)] and appended (_stratified_matrix, mcsim.py:166-180; the
// uniform draw of NONE / GLOBAL_PRESORT, :146-151, is the one-stratum case).
// out[t] is therefore the (b, G) length matrix, row-major.  Pools are not
// mutated (unlike draw_batch).  Trials are independent: `nthreads` host
// threads take contiguous trial ranges.
extern "C" int b2_mc_draw(const int32_t* lengths, const int64_t* pool_sizes, int nstrata, const int64_t* counts,
                          int num_gpus, uint64_t seed, int64_t first_trial, int64_t ntrials, int nthreads,
                          int32_t* out) {
  if (!lengths || !pool_sizes || !counts || !out || nstrata < 1 || num_gpus < 1 || ntrials < 0 || first_trial < 0) {
    b2::set_error("b2_mc_draw: bad arguments");
    return B2_ERR_INVALID;
  }
  std::vector<int64_t> off(nstrata + 1, 0);
  int64_t per_trial = 0;
  for (int k = 0; k < nstrata; ++k) {
    off[k + 1] = off[k] + pool_sizes[k];
    const int64_t need = counts[k] * (int64_t)num_gpus;
    if (counts[k] < 0 || need > pool_sizes[k]) {
      b2::set_error("corpus exhausted within a trial: a stratum holds %lld samples but the trial needs %lld",
                    (long long)pool_sizes[k], (long long)need);
      return B2_ERR_INVALID;
    }
    per_trial += need;
  }
  if (ntrials == 0) return B2_OK;
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads > 0 ? nthreads : 1, ntrials));
  auto work = [&](int64_t t0, int64_t t1) {
    std::vector<int64_t> picked, scratch;
    std::vector<uint64_t> set;
    for (int64_t t = t0; t < t1; ++t) {
      const uint64_t key = (uint64_t)(first_trial + t);
      Pcg64H rng(SeedSeq(seed, &key, 1));
      int32_t* o = out + t * per_trial;
      for (int k = 0; k < nstrata; ++k) {
        const int64_t need = counts[k] * (int64_t)num_gpus;
        if (need == 0) continue;
        rng.choice(pool_sizes[k], need, picked, scratch, set);
        const int32_t* lk = lengths + off[k];
        for (int64_t i = 0; i < need; ++i) *o++ = lk[picked[i]];
      }
    }
  };
  std::vector<std::thread> th;
  const int64_t chunk = (ntrials + nt - 1) / nt;
  for (int i = 0; i < nt; ++i) {
    const int64_t t0 = i * chunk, t1 = std::min<int64_t>(ntrials, t0 + chunk);
    if (t0 < t1) th.emplace_back(work, t0, t1);
  }
  for (auto& x : th) x.join();
  return B2_OK;
}

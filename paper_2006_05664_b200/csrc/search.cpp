// Native OpEvo proposal core (C ABI in include/opevo.h, "search" section).
//
// Restates, draw for draw, the host side of the reference's ask path so a
// generation's proposals cost microseconds instead of ~0.2 ms of Python
// (the dominant fixed cost per generation once trials are sharded over GPUs):
//   OpEvo._initial_batch / _offspring_batch   reference engine.py:228-261
//   recombine (Eq. 2)                          reference engine.py:132-147
//   mutate -> sample_walk (Eq. 3)              reference engine.py:150-157, walk.py:41-59
//   Factorization.neighbors / unrank           reference spaces.py:189-221
//   Permutation / Discrete / Categorical       reference spaces.py:266-289, 334-342, 385-387
//   uniform_index (< 2^63)                     reference spaces.py:71-84
//   Archive ranking (ties by insertion)        reference engine.py:73-116
// The random stream is numpy's Generator(PCG64) -- the RNG contract of
// PCG64 XSL-RR 128/64, random() = (u64 >> 11) * 2^-53,
// integers(n) = Lemire on buffered 32-bit halves (n <= 2^32) or on 64-bit
// draws, n == 1 consuming nothing; Generator.choice(p) = searchsorted(
// cumsum(p) / cumsum[-1], random(k), 'right') with numpy's pairwise sum.
// The caller seeds it with the numpy generator's exact state and takes it
// back for the one path left in Python (sample_unvisited, reached only when
// the retry cap is exhausted).

#include "opevo.h"

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace {

typedef unsigned __int128 u128;

struct Pcg64 {
    u128 state = 0, inc = 0;
    int has32 = 0;
    uint32_t u32 = 0;

    uint64_t next64() {
        static const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
        state = state * mult + inc;
        const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
        const unsigned rot = (unsigned)(state >> 122);
        return (x >> rot) | (x << ((-rot) & 63u));
    }
    uint32_t next32() {
        if (has32) {
            has32 = 0;
            return u32;
        }
        const uint64_t n = next64();
        has32 = 1;
        u32 = (uint32_t)(n >> 32);
        return (uint32_t)n;
    }
    double random() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
    // Generator.integers(n): uniform in [0, n)
    uint64_t integers(uint64_t n) {
        const uint64_t rng = n - 1;
        if (rng == 0) return 0;
        if (rng <= 0xFFFFFFFFull) {
            if (rng == 0xFFFFFFFFull) return next32();
            const uint32_t excl = (uint32_t)rng + 1u;
            uint64_t m = (uint64_t)next32() * excl;
            uint32_t left = (uint32_t)m;
            if (left < excl) {
                const uint32_t thresh = (UINT32_MAX - (uint32_t)rng) % excl;
                while (left < thresh) {
                    m = (uint64_t)next32() * excl;
                    left = (uint32_t)m;
                }
            }
            return m >> 32;
        }
        if (rng == UINT64_MAX) return next64();
        const uint64_t excl = rng + 1;
        u128 m = (u128)next64() * excl;
        uint64_t left = (uint64_t)m;
        if (left < excl) {
            const uint64_t thresh = (UINT64_MAX - rng) % excl;
            while (left < thresh) {
                m = (u128)next64() * excl;
                left = (uint64_t)m;
            }
        }
        return (uint64_t)(m >> 64);
    }
};

// numpy's float64 add.reduce over a contiguous array (pairwise summation)
double np_sum(const double* a, size_t n) {
    if (n < 8) {
        double r = 0.0;
        for (size_t i = 0; i < n; ++i) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        size_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    size_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_sum(a, n2) + np_sum(a + n2, n - n2);
}

typedef std::vector<int64_t> Tup;

struct TupHash {
    size_t operator()(const Tup& t) const {
        uint64_t h = 1469598103934665603ull;
        for (int64_t v : t) {
            h ^= (uint64_t)v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
            h *= 1099511628211ull;
        }
        return (size_t)h;
    }
};

uint64_t binom(uint64_t n, uint64_t k) {
    if (k > n) return 0;
    uint64_t r = 1;
    for (uint64_t i = 1; i <= k; ++i) r = r * (n - k + i) / i;
    return r;
}

std::vector<std::pair<int64_t, int>> factorize(int64_t n) {
    std::vector<std::pair<int64_t, int>> out;
    for (int64_t p = 2; p * p <= n; p += (p == 2 ? 1 : 2)) {
        int e = 0;
        while (n % p == 0) {
            n /= p;
            ++e;
        }
        if (e) out.push_back({p, e});
    }
    if (n > 1) out.push_back({n, 1});
    return out;
}

// One parameter of the product space.  Values are interned: a config holds
// one id per parameter (index into `vals`); a value's slot form is the tuple
// (factorization, permutation) or {index} (discrete, categorical).
struct Param {
    int kind = 0;            // OPEVO_PARAM_*
    int64_t a = 0;           // factorization product / discrete, categorical count / permutation items
    int arity = 1;           // slots of the value
    uint64_t size = 0;
    std::vector<std::pair<int64_t, int>> primes;          // factorization
    std::vector<Tup> vals;                                // interned values (slot form)
    std::unordered_map<Tup, int, TupHash> ids;
    std::vector<std::vector<int>> nbrs;                   // per id, canonical order
    std::vector<char> have_nbrs;

    int intern(const Tup& t) {
        auto it = ids.find(t);
        if (it != ids.end()) return it->second;
        const int id = (int)vals.size();
        vals.push_back(t);
        ids.emplace(t, id);
        nbrs.emplace_back();
        have_nbrs.push_back(0);
        return id;
    }

    uint64_t completions(int64_t rest, int slots) const {
        uint64_t c = 1;
        for (auto& pe : factorize(rest)) c *= binom((uint64_t)pe.second + slots - 1, (uint64_t)slots - 1);
        return c;
    }

    // the canonical enumeration's index-th value
    Tup unrank(uint64_t index) const {
        Tup out;
        if (kind == OPEVO_PARAM_FACTORIZATION) {
            int64_t left = a;
            for (int after = arity - 1; after >= 1; --after) {
                std::vector<int64_t> divs;
                for (int64_t d = 1; d * d <= left; ++d)
                    if (left % d == 0) {
                        divs.push_back(d);
                        if (d != left / d) divs.push_back(left / d);
                    }
                std::sort(divs.begin(), divs.end());
                for (int64_t d : divs) {
                    const uint64_t block = completions(left / d, after);
                    if (index < block) {
                        out.push_back(d);
                        left /= d;
                        break;
                    }
                    index -= block;
                }
            }
            out.push_back(left);
        } else if (kind == OPEVO_PARAM_PERMUTATION) {
            std::vector<int64_t> pool;
            for (int64_t i = 0; i < a; ++i) pool.push_back(i);
            for (int64_t remaining = a; remaining >= 1; --remaining) {
                uint64_t block = 1;
                for (int64_t f = 2; f <= remaining - 1; ++f) block *= (uint64_t)f;
                const uint64_t digit = index / block;
                index %= block;
                out.push_back(pool[digit]);
                pool.erase(pool.begin() + (long)digit);
            }
        } else {
            out.push_back((int64_t)index);
        }
        return out;
    }

    const std::vector<int>& neighbors(int id) {
        if (have_nbrs[id]) return nbrs[id];
        const Tup v = vals[id];
        std::vector<Tup> out;
        if (kind == OPEVO_PARAM_FACTORIZATION) {
            for (auto& pe : primes) {
                const int64_t p = pe.first;
                for (int src = 0; src < arity; ++src) {
                    if (v[src] % p) continue;
                    for (int dst = 0; dst < arity; ++dst) {
                        if (dst == src) continue;
                        Tup w = v;
                        w[src] /= p;
                        w[dst] *= p;
                        out.push_back(w);
                    }
                }
            }
            std::sort(out.begin(), out.end());
            out.erase(std::unique(out.begin(), out.end()), out.end());
        } else if (kind == OPEVO_PARAM_PERMUTATION) {
            for (int i = 0; i < arity; ++i)
                for (int j = i + 1; j < arity; ++j) {
                    Tup w = v;
                    std::swap(w[i], w[j]);
                    out.push_back(w);
                }
            std::sort(out.begin(), out.end());
        } else if (kind == OPEVO_PARAM_DISCRETE) {
            if (v[0] - 1 >= 0) out.push_back(Tup{v[0] - 1});
            if (v[0] + 1 < a) out.push_back(Tup{v[0] + 1});
        } else {
            for (int64_t x = 0; x < a; ++x)
                if (x != v[0]) out.push_back(Tup{x});
        }
        std::vector<int> ids_out;
        ids_out.reserve(out.size());
        for (auto& w : out) ids_out.push_back(intern(w));
        // intern() may have grown the tables: index afresh
        nbrs[id] = std::move(ids_out);
        have_nbrs[id] = 1;
        return nbrs[id];
    }
};

struct Member {
    std::vector<int> cfg;
    double fitness;
};

struct CfgHash {
    size_t operator()(const std::vector<int>& v) const {
        uint64_t h = 1469598103934665603ull;
        for (int x : v) {
            h ^= (uint64_t)(uint32_t)x;
            h *= 1099511628211ull;
        }
        return (size_t)h;
    }
};

}  // namespace

struct opevo_search {
    std::vector<Param> params;
    int slots = 0;
    int parents = 8, offspring = 8, retry_cap = 64;
    double q = 0.5;
    Pcg64 rng;
    // archive: ranked by -fitness ascending, ties by insertion (bisect_right)
    std::vector<double> keys;
    std::vector<int> ranked;                     // indices into members
    std::vector<Member> members;
    std::unordered_set<std::vector<int>, CfgHash> visited;   // archive configs
    // the pending batch (in ask order) and its set
    std::vector<std::vector<int>> batch;
    std::unordered_set<std::vector<int>, CfgHash> chosen;
};

namespace {

void to_slots(opevo_search* s, const std::vector<int>& cfg, int64_t* out) {
    int o = 0;
    for (size_t i = 0; i < s->params.size(); ++i) {
        const Tup& v = s->params[i].vals[cfg[i]];
        for (int64_t x : v) out[o++] = x;
    }
}

bool from_slots(opevo_search* s, const int64_t* in, std::vector<int>& cfg) {
    cfg.resize(s->params.size());
    int o = 0;
    for (size_t i = 0; i < s->params.size(); ++i) {
        Param& p = s->params[i];
        Tup t(in + o, in + o + p.arity);
        o += p.arity;
        cfg[i] = p.intern(t);
    }
    return true;
}

std::vector<int> sample_uniform(opevo_search* s) {
    std::vector<int> cfg(s->params.size());
    for (size_t i = 0; i < s->params.size(); ++i) {
        Param& p = s->params[i];
        cfg[i] = p.intern(p.unrank(s->rng.integers(p.size)));
    }
    return cfg;
}

std::vector<int> recombine(opevo_search* s, const std::vector<int>& par) {
    const size_t n = par.size(), k = s->params.size();
    std::vector<double> fit(n);
    for (size_t j = 0; j < n; ++j) fit[j] = s->members[par[j]].fitness;
    const double total = np_sum(fit.data(), n);
    std::vector<size_t> donor(k);
    if (total > 0.0) {
        std::vector<double> cdf(n);
        double acc = 0.0;
        for (size_t j = 0; j < n; ++j) {
            acc += fit[j] / total;
            cdf[j] = acc;
        }
        const double last = cdf[n - 1];
        for (size_t j = 0; j < n; ++j) cdf[j] /= last;
        for (size_t i = 0; i < k; ++i) {
            const double u = s->rng.random();
            donor[i] = (size_t)(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
        }
    } else {
        for (size_t i = 0; i < k; ++i) donor[i] = (size_t)s->rng.integers(n);
    }
    std::vector<int> child(k);
    for (size_t i = 0; i < k; ++i) child[i] = s->members[par[donor[i]]].cfg[i];
    return child;
}

int walk(opevo_search* s, Param& p, int here) {
    for (int steps = 0; steps < 1000000; ++steps) {
        if (s->rng.random() >= s->q) return here;
        const std::vector<int>& nb = p.neighbors(here);
        if (nb.empty()) return here;
        here = nb[(size_t)s->rng.integers(nb.size())];
    }
    return -1;
}

}  // namespace

extern "C" {

int opevo_search_create(int nparams, const int32_t* kinds, const int64_t* a, const int32_t* arity,
                        int parents, int offspring, double q, int retry_cap, opevo_search** out) {
    if (!out || nparams < 1 || !kinds || !a || parents < 1 || offspring < 1 || retry_cap < 1 ||
        !(q >= 0.0 && q < 1.0))
        return OPEVO_ERR_ARG;
    opevo_search* s = new opevo_search();
    s->parents = parents;
    s->offspring = offspring;
    s->q = q;
    s->retry_cap = retry_cap;
    for (int i = 0; i < nparams; ++i) {
        Param p;
        p.kind = kinds[i];
        p.a = a[i];
        if (p.a < 1) {
            delete s;
            return OPEVO_ERR_ARG;
        }
        if (p.kind == OPEVO_PARAM_FACTORIZATION) {
            p.arity = arity ? arity[i] : 1;
            if (p.arity < 1) {
                delete s;
                return OPEVO_ERR_ARG;
            }
            p.primes = factorize(p.a);
            p.size = 1;
            for (auto& pe : p.primes) p.size *= binom((uint64_t)pe.second + p.arity - 1, (uint64_t)p.arity - 1);
        } else if (p.kind == OPEVO_PARAM_PERMUTATION) {
            p.arity = (int)p.a;
            if (p.a > 20) {            // 21! exceeds 2^63: the reference draws bytes there
                delete s;
                return OPEVO_ERR_ARG;
            }
            p.size = 1;
            for (int64_t f = 2; f <= p.a; ++f) p.size *= (uint64_t)f;
        } else if (p.kind == OPEVO_PARAM_DISCRETE || p.kind == OPEVO_PARAM_CATEGORICAL) {
            p.size = (uint64_t)p.a;
        } else {
            delete s;
            return OPEVO_ERR_ARG;
        }
        s->slots += p.arity;
        s->params.push_back(std::move(p));
    }
    *out = s;
    return OPEVO_OK;
}

void opevo_search_destroy(opevo_search* s) { delete s; }

int opevo_search_slots(const opevo_search* s) { return s ? s->slots : OPEVO_ERR_ARG; }

int opevo_search_set_rng(opevo_search* s, const uint64_t st[4], int has_uint32, uint32_t uinteger) {
    if (!s || !st) return OPEVO_ERR_ARG;
    s->rng.state = ((u128)st[0] << 64) | (u128)st[1];
    s->rng.inc = ((u128)st[2] << 64) | (u128)st[3];
    s->rng.has32 = has_uint32 ? 1 : 0;
    s->rng.u32 = uinteger;
    return OPEVO_OK;
}

int opevo_search_get_rng(const opevo_search* s, uint64_t st[4], int* has_uint32, uint32_t* uinteger) {
    if (!s || !st) return OPEVO_ERR_ARG;
    st[0] = (uint64_t)(s->rng.state >> 64);
    st[1] = (uint64_t)s->rng.state;
    st[2] = (uint64_t)(s->rng.inc >> 64);
    st[3] = (uint64_t)s->rng.inc;
    if (has_uint32) *has_uint32 = s->rng.has32;
    if (uinteger) *uinteger = s->rng.u32;
    return OPEVO_OK;
}

int opevo_search_propose(opevo_search* s, int initial, int first, int want, int64_t* out,
                         int* need_fallback) {
    if (!s || want < 0 || (want > 0 && !out) || !need_fallback) return OPEVO_ERR_ARG;
    *need_fallback = 0;
    if (first) {
        s->batch.clear();
        s->chosen.clear();
    }
    std::vector<int> par;
    if (!initial) {
        if (s->ranked.empty()) return OPEVO_ERR_ARG;
        const size_t np_ = std::min(s->ranked.size(), (size_t)s->parents);
        par.assign(s->ranked.begin(), s->ranked.begin() + (long)np_);
    }
    int made = 0;
    for (; made < want; ++made) {
        bool ok = false;
        std::vector<int> pick;
        if (initial) {
            for (int r = 0; r < s->retry_cap && !ok; ++r) {
                pick = sample_uniform(s);
                ok = !s->chosen.count(pick);
            }
        } else {
            const std::vector<int> base = recombine(s, par);
            for (int r = 0; r < s->retry_cap && !ok; ++r) {
                pick = base;
                for (size_t i = 0; i < pick.size(); ++i) {
                    pick[i] = walk(s, s->params[i], pick[i]);
                    if (pick[i] < 0) return OPEVO_SEARCH_WALK_LIMIT;   // the reference raises RuntimeError
                }
                ok = !s->visited.count(pick) && !s->chosen.count(pick);
            }
        }
        if (!ok) {
            *need_fallback = 1;       // sample_unvisited: the caller draws it with this RNG state
            break;
        }
        to_slots(s, pick, out + (size_t)made * s->slots);
        s->chosen.insert(pick);
        s->batch.push_back(std::move(pick));
    }
    return made;
}

int opevo_search_add_pending(opevo_search* s, const int64_t* slots) {
    if (!s || !slots) return OPEVO_ERR_ARG;
    std::vector<int> cfg;
    from_slots(s, slots, cfg);
    s->chosen.insert(cfg);
    s->batch.push_back(std::move(cfg));
    return OPEVO_OK;
}

int opevo_search_tell(opevo_search* s, int n, const int64_t* slots, const double* fitness) {
    if (!s || n < 0 || (n > 0 && (!slots || !fitness))) return OPEVO_ERR_ARG;
    for (int i = 0; i < n; ++i) {
        std::vector<int> cfg;
        from_slots(s, slots + (size_t)i * s->slots, cfg);
        if (s->visited.count(cfg)) return OPEVO_ERR_ARG;
        const double key = -fitness[i];
        const size_t pos = (size_t)(std::upper_bound(s->keys.begin(), s->keys.end(), key) - s->keys.begin());
        s->keys.insert(s->keys.begin() + (long)pos, key);
        s->ranked.insert(s->ranked.begin() + (long)pos, (int)s->members.size());
        s->visited.insert(cfg);
        s->members.push_back(Member{std::move(cfg), fitness[i]});
    }
    s->batch.clear();
    s->chosen.clear();
    return OPEVO_OK;
}

int opevo_search_uniform_int(opevo_search* s, uint64_t n, uint64_t* out) {
    if (!s || !out || n == 0) return OPEVO_ERR_ARG;
    *out = s->rng.integers(n);
    return OPEVO_OK;
}

int opevo_search_random(opevo_search* s, double* out) {
    if (!s || !out) return OPEVO_ERR_ARG;
    *out = s->rng.random();
    return OPEVO_OK;
}

double opevo_search_np_sum(const double* a, size_t n) { return np_sum(a, n); }

}  // extern "C"

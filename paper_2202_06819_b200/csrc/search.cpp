// search.cpp -- learned, diversity-aware schedule search.
//
// Host-only C++ (no CUDA): the exploration module of PAPER.md section 3.4
// with the settings of section 4.1,
// over a generic knob space.  conv_q_plan_search (convq.cu) instantiates it
// with the conv plan's TileConfig knobs + runtime knobs and device timing;
// tests/test_search_cpu.py drives conv_q_search with synthetic cost functions.
//
//   * cost model: "trained by {(configuration, runtime)} dataset
//     with ranking loss objective" -- here a linear scorer over one-hot knob
//     features and all pairwise knob crosses, trained with the pairwise
//     logistic (RankNet) loss; higher score = predicted faster (DESIGN reading 17);
//   * simulated annealing: parallel chains (128), "mutate one
//     random knob", energy = the model score, acceptance exp(min((s'-s)/T, 1)),
//     T starts at 1 and cools by 0.002 per iteration, 500 iterations, stop when
//     the optimal set has not changed for 50 iterations; only never-measured
//     points enter the optimal set;
//   * diversity-aware selection: each chain's point makes TWO
//     mutants, half of all mutants are kept by configuration diversity (greedy
//     farthest-point in Hamming distance, seeded with the best-scored mutant),
//     and each kept mutant competes with its parent (DESIGN reading 18);
//   * measurement batches: the top (batch - 1) = 31 points of
//     the optimal set plus one random never-measured point are measured; fewer
//     than 31 new candidates -> random points fill the rest; the measurements
//     retrain the model.  The first batch is random (no model yet).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <unordered_map>
#include <unordered_set>
#include <utility>
#include <vector>

#include "../../include/convq.h"

namespace convq {
int set_err(int code, const char *fmt, ...);
}

namespace {

struct Rng {   // splitmix64: deterministic for a seed on every platform
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    int below(int n) { return (int)(next() % (uint64_t)n); }
    double uniform() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

struct Space {
    int n;
    std::vector<int> sizes;
    conv_q_valid_fn valid;
    void *ctx;
    uint64_t key(const int *k) const {   // mixed-radix index of a point
        uint64_t v = 0;
        for (int i = 0; i < n; ++i) v = v * (uint64_t)sizes[i] + (uint64_t)k[i];
        return v;
    }
    bool ok(const int *k) const { return !valid || valid(ctx, k) != 0; }
};

// Linear scorer over one-hot knob values + one-hot pairwise crosses.
struct RankModel {
    const Space *sp;
    std::vector<int> off1;                 // one-hot offset of knob i
    std::vector<std::vector<int>> off2;    // cross offset of knob pair (i < j)
    int dim = 0;
    std::vector<double> w;
    explicit RankModel(const Space *s) : sp(s) {
        off1.resize(s->n);
        for (int i = 0; i < s->n; ++i) { off1[i] = dim; dim += s->sizes[i]; }
        off2.assign(s->n, std::vector<int>(s->n, -1));
        for (int i = 0; i < s->n; ++i)
            for (int j = i + 1; j < s->n; ++j) { off2[i][j] = dim; dim += s->sizes[i] * s->sizes[j]; }
        w.assign(dim, 0.0);
    }
    void features(const int *k, std::vector<int> &f) const {
        f.clear();
        for (int i = 0; i < sp->n; ++i) f.push_back(off1[i] + k[i]);
        for (int i = 0; i < sp->n; ++i)
            for (int j = i + 1; j < sp->n; ++j) f.push_back(off2[i][j] + k[i] * sp->sizes[j] + k[j]);
    }
    double score(const int *k) const {
        double s = 0;
        for (int i = 0; i < sp->n; ++i) s += w[off1[i] + k[i]];
        for (int i = 0; i < sp->n; ++i)
            for (int j = i + 1; j < sp->n; ++j) s += w[off2[i][j] + k[i] * sp->sizes[j] + k[j]];
        return s;
    }
    // RankNet: for a pair with cost_a < cost_b, loss = log(1 + exp(-(s_a - s_b))).
    // Failed measurements rank below every successful one.  Full re-fit from
    // zero after every batch (the dataset is small: <= a few hundred points).
    void fit(const std::vector<std::vector<int>> &X, const std::vector<double> &cost, Rng &rng) {
        std::fill(w.begin(), w.end(), 0.0);
        const int n = (int)X.size();
        if (n < 2) return;
        std::vector<std::vector<int>> F(n);
        for (int i = 0; i < n; ++i) features(X[i].data(), F[i]);
        auto rank_cost = [&](int i) { return cost[i] > 0 ? cost[i] : std::numeric_limits<double>::infinity(); };
        const int epochs = 60;
        const int pairs = std::min(4000, n * (n - 1) / 2 * 2);
        const double lr = 0.1, l2 = 1e-4;
        for (int e = 0; e < epochs; ++e) {
            const double rate = lr / (1.0 + 0.05 * e);
            for (int t = 0; t < pairs; ++t) {
                int a = rng.below(n), b = rng.below(n);
                double ca = rank_cost(a), cb = rank_cost(b);
                if (a == b || ca == cb) continue;
                if (ca > cb) std::swap(a, b);   // a is the faster one
                double sa = 0, sb = 0;
                for (int f : F[a]) sa += w[f];
                for (int f : F[b]) sb += w[f];
                const double d = sa - sb;
                const double gr = 1.0 / (1.0 + std::exp(d));   // -dloss/dd
                for (int f : F[a]) w[f] += rate * (gr - l2 * w[f]);
                for (int f : F[b]) w[f] -= rate * (gr + l2 * w[f]);
            }
        }
    }
};

int hamming(const std::vector<int> &a, const std::vector<int> &b) {
    int d = 0;
    for (size_t i = 0; i < a.size(); ++i) d += a[i] != b[i];
    return d;
}

// a random valid point (rejection sampling; false if none found)
bool random_point(const Space &sp, Rng &rng, std::vector<int> &k) {
    k.assign(sp.n, 0);
    for (int t = 0; t < 100000; ++t) {
        for (int i = 0; i < sp.n; ++i) k[i] = rng.below(sp.sizes[i]);
        if (sp.ok(k.data())) return true;
    }
    return false;
}

// "mutate one random knob": a different value of one knob, valid
bool mutate(const Space &sp, Rng &rng, const std::vector<int> &from, std::vector<int> &to) {
    to = from;
    for (int t = 0; t < 32; ++t) {
        const int i = rng.below(sp.n);
        if (sp.sizes[i] < 2) continue;
        to = from;
        to[i] = (from[i] + 1 + rng.below(sp.sizes[i] - 1)) % sp.sizes[i];
        if (sp.ok(to.data())) return true;
    }
    to = from;
    return false;
}

// Simulated annealing over the model score; returns up to `want` never-measured
// points with the best scores seen (the "optimal set").
std::vector<std::vector<int>> sa_pick(const Space &sp, const RankModel &m, const conv_q_search_opts_t &o,
                                      const std::unordered_set<uint64_t> &measured,
                                      const std::vector<std::vector<int>> &seeds, int want, Rng &rng) {
    const int npts = std::max(1, o.sa_points);
    std::vector<std::vector<int>> pts;
    // start from the best measured points, then random ones (AutoTVM keeps its previous chains)
    for (size_t i = 0; i < seeds.size() && (int)pts.size() < npts / 2; ++i) pts.push_back(seeds[i]);
    std::vector<int> k;
    while ((int)pts.size() < npts && random_point(sp, rng, k)) pts.push_back(k);
    std::vector<double> sc(pts.size());
    for (size_t i = 0; i < pts.size(); ++i) sc[i] = m.score(pts[i].data());
    // optimal set: (score, key) of the best `want` unmeasured points seen
    std::vector<std::pair<double, uint64_t>> best;
    std::unordered_map<uint64_t, std::vector<int>> best_pts;
    auto offer = [&](const std::vector<int> &p, double s) -> bool {
        const uint64_t key = sp.key(p.data());
        if (measured.count(key) || best_pts.count(key)) return false;
        if ((int)best.size() < want) {
            best.push_back({s, key});
            best_pts[key] = p;
            return true;
        }
        auto worst = std::min_element(best.begin(), best.end());
        if (s <= worst->first) return false;
        best_pts.erase(worst->second);
        *worst = {s, key};
        best_pts[key] = p;
        return true;
    };
    for (size_t i = 0; i < pts.size(); ++i) offer(pts[i], sc[i]);
    double T = o.sa_temp0;
    int last_change = 0;
    std::vector<int> mu;
    for (int it = 0; it < o.sa_iters && it < last_change + o.sa_early_stop; ++it) {
        const int n = (int)pts.size();
        std::vector<std::vector<int>> cand(n);
        std::vector<double> cs(n);
        std::vector<char> has(n, 0);
        if (o.diversity) {
            // two mutants per parent; keep half of all mutants by diversity
            std::vector<std::vector<int>> mut;
            std::vector<int> parent;
            std::vector<double> ms;
            for (int i = 0; i < n; ++i)
                for (int r = 0; r < 2; ++r)
                    if (mutate(sp, rng, pts[i], mu)) {
                        mut.push_back(mu);
                        parent.push_back(i);
                        ms.push_back(m.score(mu.data()));
                    }
            const int nm = (int)mut.size(), keep = nm / 2;
            std::vector<char> sel(nm, 0);
            std::vector<int> mind(nm, std::numeric_limits<int>::max());
            int first = -1;
            for (int i = 0; i < nm; ++i)
                if (first < 0 || ms[i] > ms[first]) first = i;
            for (int c = 0, pick = first; c < keep && pick >= 0; ++c) {
                sel[pick] = 1;
                for (int i = 0; i < nm; ++i) mind[i] = std::min(mind[i], hamming(mut[i], mut[pick]));
                pick = -1;
                for (int i = 0; i < nm; ++i)
                    if (!sel[i] && (pick < 0 || mind[i] > mind[pick] || (mind[i] == mind[pick] && ms[i] > ms[pick])))
                        pick = i;
            }
            // each kept mutant competes with its parent (a parent with two kept
            // mutants: the better-scored one)
            for (int i = 0; i < nm; ++i)
                if (sel[i] && (!has[parent[i]] || ms[i] > cs[parent[i]])) {
                    cand[parent[i]] = mut[i];
                    cs[parent[i]] = ms[i];
                    has[parent[i]] = 1;
                }
        } else {
            for (int i = 0; i < n; ++i)
                if (mutate(sp, rng, pts[i], mu)) {
                    cand[i] = mu;
                    cs[i] = m.score(mu.data());
                    has[i] = 1;
                }
        }
        bool changed = false;
        for (int i = 0; i < n; ++i) {
            if (!has[i]) continue;
            changed |= offer(cand[i], cs[i]);
            const double ac = std::exp(std::min((cs[i] - sc[i]) / (T + 1e-5), 1.0));
            if (rng.uniform() < ac) {
                pts[i] = cand[i];
                sc[i] = cs[i];
            }
        }
        if (changed) last_change = it;
        T = std::max(T - (double)o.sa_cool, 0.0);
    }
    std::sort(best.begin(), best.end(), [](const std::pair<double, uint64_t> &a, const std::pair<double, uint64_t> &b) {
        return a.first > b.first || (a.first == b.first && a.second < b.second);
    });
    std::vector<std::vector<int>> out;
    for (auto &b : best) out.push_back(best_pts[b.second]);
    return out;
}

}  // namespace

extern "C" void conv_q_search_opts_default(conv_q_search_opts_t *o) {
    if (!o) return;
    o->trials = 128;
    o->batch = 32;          // 31 model picks + 1 random
    o->sa_iters = 500;
    o->sa_early_stop = 50;
    o->sa_points = 128;
    o->diversity = 1;
    o->sa_temp0 = 1.0f;
    o->sa_cool = 0.002f;
    o->seed = 6819;
}

extern "C" int conv_q_search(int n_knobs, const int *knob_sizes, conv_q_valid_fn valid, conv_q_cost_fn cost, void *ctx,
                             const conv_q_search_opts_t *opts, int *best_knobs, double *history_cost,
                             int *history_knobs) {
    using convq::set_err;
    if (n_knobs < 1 || n_knobs > CONV_Q_SEARCH_MAX_KNOBS || !knob_sizes || !cost || !best_knobs)
        return set_err(CONV_Q_EINVAL, "conv_q_search: bad arguments");
    conv_q_search_opts_t o;
    conv_q_search_opts_default(&o);
    if (opts) o = *opts;
    if (o.trials < 1 || o.batch < 1 || o.sa_points < 1 || o.sa_iters < 0 || o.sa_early_stop < 1)
        return set_err(CONV_Q_EINVAL, "conv_q_search: trials, batch, sa_points, sa_early_stop >= 1, sa_iters >= 0");
    Space sp{n_knobs, std::vector<int>(knob_sizes, knob_sizes + n_knobs), valid, ctx};
    double total = 1;
    for (int s : sp.sizes) {
        if (s < 1) return set_err(CONV_Q_EINVAL, "conv_q_search: knob sizes must be >= 1");
        total *= s;
    }
    if (total > 1e18) return set_err(CONV_Q_EINVAL, "conv_q_search: space too large for 64-bit point keys");
    Rng rng(o.seed);
    RankModel model(&sp);
    std::vector<std::vector<int>> X;
    std::vector<double> Y;
    std::unordered_set<uint64_t> measured;
    int best = -1;
    std::vector<int> k;
    auto measure = [&](const std::vector<int> &p) {
        const double c = cost(ctx, p.data());
        if (history_cost) history_cost[X.size()] = c;
        if (history_knobs) std::memcpy(history_knobs + X.size() * n_knobs, p.data(), sizeof(int) * n_knobs);
        measured.insert(sp.key(p.data()));
        X.push_back(p);
        Y.push_back(c);
        if (c > 0 && (best < 0 || c < Y[best])) best = (int)X.size() - 1;
    };
    auto random_new = [&](std::vector<int> &p) {
        for (int t = 0; t < 1000; ++t) {
            if (!random_point(sp, rng, p)) return false;
            if (!measured.count(sp.key(p.data()))) return true;
        }
        return false;
    };
    bool exhausted = false;
    while ((int)X.size() < o.trials && !exhausted) {
        const int room = std::min(o.batch, o.trials - (int)X.size());
        std::vector<std::vector<int>> batch;
        if (!X.empty()) {
            model.fit(X, Y, rng);
            // chains seeded from the best measured points
            std::vector<int> order(X.size());
            for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
            std::sort(order.begin(), order.end(), [&](int a, int b) {
                const double ca = Y[a] > 0 ? Y[a] : 1e300, cb = Y[b] > 0 ? Y[b] : 1e300;
                return ca < cb || (ca == cb && a < b);
            });
            std::vector<std::vector<int>> seeds;
            for (int i = 0; i < (int)order.size() && i < 16; ++i)
                if (Y[order[i]] > 0) seeds.push_back(X[order[i]]);
            batch = sa_pick(sp, model, o, measured, seeds, std::max(room - 1, 1), rng);
            if ((int)batch.size() > room - 1 && room > 1) batch.resize(room - 1);
            if (room == 1 && !batch.empty()) batch.resize(1);
        }
        // + one random point, and random fill when the model found too few new points
        std::unordered_set<uint64_t> inb;
        for (auto &b : batch) inb.insert(sp.key(b.data()));
        while ((int)batch.size() < room) {
            bool found = false;
            for (int t = 0; t < 64 && !found; ++t)
                if (random_new(k) && !inb.count(sp.key(k.data()))) found = true;
            if (!found) {
                exhausted = batch.empty();
                break;
            }
            inb.insert(sp.key(k.data()));
            batch.push_back(k);
        }
        for (auto &b : batch) measure(b);
    }
    if (best < 0) return set_err(CONV_Q_ECUDA, "conv_q_search: no point measured successfully");
    std::memcpy(best_knobs, X[best].data(), sizeof(int) * n_knobs);
    return (int)X.size();
}

// Seeded synthetic graph generators for the benchmark shapes of BASELINE.json
// (planted-partition SBM, LFR-style power-law communities, R-MAT). Workload
// infrastructure for bench.py and the tests, not part of the product path.
//
// Every generator returns the CSR that graphqc::Graph(n, edges, W) would
// build (graph.cpp:25-71): undirected, no self loops, duplicates collapsed,
// neighbour ids ascending per row, unit weights. Deterministic for a seed.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

namespace {

struct Rng {  // splitmix64
    std::uint64_t s;
    explicit Rng(std::uint64_t seed) : s(seed) {}
    std::uint64_t next() {
        std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform() { return (next() >> 11) * 0x1.0p-53; }
    std::uint64_t below(std::uint64_t n) { return static_cast<std::uint64_t>(uniform() * n) % n; }
};

struct Csr {
    std::vector<std::int64_t> offsets;
    std::vector<std::int32_t> nbr;
};

// Undirected edge list -> CSR with dedup and ascending rows (counting sort by
// row, then sort + unique inside each row).
Csr build_csr(std::int32_t n, const std::vector<std::pair<std::int32_t, std::int32_t>>& edges) {
    std::vector<std::int64_t> deg(n + 1, 0);
    for (auto [u, v] : edges) {
        if (u == v) continue;
        ++deg[u + 1];
        ++deg[v + 1];
    }
    for (std::int32_t i = 0; i < n; ++i) deg[i + 1] += deg[i];
    std::vector<std::int32_t> tmp(deg[n]);
    std::vector<std::int64_t> cur(deg.begin(), deg.end() - 1);
    for (auto [u, v] : edges) {
        if (u == v) continue;
        tmp[cur[u]++] = v;
        tmp[cur[v]++] = u;
    }
    Csr g;
    g.offsets.assign(n + 1, 0);
    g.nbr.reserve(tmp.size());
    for (std::int32_t i = 0; i < n; ++i) {
        auto b = tmp.begin() + deg[i], e = tmp.begin() + deg[i + 1];
        std::sort(b, e);
        auto last = std::unique(b, e);
        g.nbr.insert(g.nbr.end(), b, last);
        g.offsets[i + 1] = static_cast<std::int64_t>(g.nbr.size());
    }
    return g;
}

// Planted partition: `blocks` blocks of `size` consecutive ids; round(n*deg/2)
// edge draws, a fraction `intra` inside a uniformly chosen block.
thread_local std::vector<std::int32_t> g_labels;  // planted communities of the last graph

Csr sbm(std::int32_t blocks, std::int32_t size, double avg_deg, double intra, std::uint64_t seed) {
    Rng r(seed);
    const std::int32_t n = blocks * size;
    g_labels.resize(n);
    for (std::int32_t i = 0; i < n; ++i) g_labels[i] = i / size;
    const std::int64_t m = std::llround(n * avg_deg / 2.0);
    std::vector<std::pair<std::int32_t, std::int32_t>> e;
    e.reserve(m);
    for (std::int64_t t = 0; t < m; ++t) {
        if (r.uniform() < intra) {
            const std::int32_t b = static_cast<std::int32_t>(r.below(blocks));
            e.emplace_back(b * size + static_cast<std::int32_t>(r.below(size)),
                           b * size + static_cast<std::int32_t>(r.below(size)));
        } else {
            std::int32_t u = static_cast<std::int32_t>(r.below(n)), v;
            do v = static_cast<std::int32_t>(r.below(n)); while (v / size == u / size);
            e.emplace_back(u, v);
        }
    }
    return build_csr(n, e);
}

// Continuous power law x^-tau on [lo, hi], inverse-CDF sample.
double power_law(Rng& r, double tau, double lo, double hi) {
    const double a = 1.0 - tau;
    const double u = r.uniform();
    return std::pow(std::pow(lo, a) + u * (std::pow(hi, a) - std::pow(lo, a)), 1.0 / a);
}

// LFR-style benchmark (configuration model): power-law degrees (tau1, kmax)
// with kmin chosen for the requested mean, power-law community sizes (tau2,
// [cmin, cmax]), mixing mu: a fraction (1-mu) of each node's stubs is paired
// inside its community, the rest across the graph. Node ids are a random
// permutation of the community layout.
Csr lfr(std::int32_t n, double avg_deg, double tau1, double kmax, double tau2, double cmin, double cmax, double mu,
        std::uint64_t seed) {
    Rng r(seed);
    // kmin by bisection on the continuous mean
    auto mean_of = [&](double kmin) {
        const double a = 1.0 - tau1, b = 2.0 - tau1;
        return (a / b) * (std::pow(kmax, b) - std::pow(kmin, b)) / (std::pow(kmax, a) - std::pow(kmin, a));
    };
    double lo = 1.0, hi = kmax;
    for (int it = 0; it < 100; ++it) {
        const double mid = 0.5 * (lo + hi);
        (mean_of(mid) < avg_deg ? lo : hi) = mid;
    }
    const double kmin = 0.5 * (lo + hi);
    std::vector<std::int32_t> deg(n);
    for (auto& d : deg) d = static_cast<std::int32_t>(std::llround(power_law(r, tau1, kmin, kmax)));
    // communities
    std::vector<std::int32_t> sizes;
    std::int64_t total = 0;
    while (total < n) {
        std::int32_t s = static_cast<std::int32_t>(std::llround(power_law(r, tau2, cmin, cmax)));
        if (total + s > n) s = static_cast<std::int32_t>(n - total);
        sizes.push_back(s);
        total += s;
    }
    std::vector<std::int32_t> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    for (std::int32_t i = n - 1; i > 0; --i) std::swap(perm[i], perm[r.below(i + 1)]);
    std::vector<std::pair<std::int32_t, std::int32_t>> e;
    e.reserve(static_cast<std::size_t>(n * avg_deg / 2 * 1.05));
    std::vector<std::int32_t> ext_stubs;
    std::int64_t base = 0;
    std::vector<std::int32_t> stubs;
    g_labels.assign(n, 0);
    std::int32_t community = 0;
    for (std::int32_t sz : sizes) {
        for (std::int32_t t = 0; t < sz; ++t) g_labels[perm[base + t]] = community;
        ++community;
        stubs.clear();
        for (std::int32_t t = 0; t < sz; ++t) {
            const std::int32_t node = perm[base + t];
            std::int32_t kin = static_cast<std::int32_t>(std::llround((1.0 - mu) * deg[node]));
            kin = std::min(kin, sz - 1);
            for (std::int32_t q = 0; q < kin; ++q) stubs.push_back(node);
            for (std::int32_t q = kin; q < deg[node]; ++q) ext_stubs.push_back(node);
        }
        for (std::size_t i = stubs.size(); i > 1; --i) std::swap(stubs[i - 1], stubs[r.below(i)]);
        for (std::size_t i = 0; i + 1 < stubs.size(); i += 2) e.emplace_back(stubs[i], stubs[i + 1]);
        base += sz;
    }
    for (std::size_t i = ext_stubs.size(); i > 1; --i) std::swap(ext_stubs[i - 1], ext_stubs[r.below(i)]);
    for (std::size_t i = 0; i + 1 < ext_stubs.size(); i += 2) e.emplace_back(ext_stubs[i], ext_stubs[i + 1]);
    return build_csr(n, e);
}

// R-MAT (Chakrabarti et al.): 2^scale nodes, edge_factor * 2^scale edge draws,
// quadrant probabilities (a, b, c, 1-a-b-c).
Csr rmat(int scale, double edge_factor, double a, double b, double c, std::uint64_t seed) {
    Rng r(seed);
    const std::int32_t n = 1 << scale;
    g_labels.clear();  // no planted partition
    const std::int64_t m = static_cast<std::int64_t>(edge_factor * n);
    std::vector<std::pair<std::int32_t, std::int32_t>> e;
    e.reserve(m);
    for (std::int64_t t = 0; t < m; ++t) {
        std::int32_t u = 0, v = 0;
        for (int bit = scale - 1; bit >= 0; --bit) {
            const double x = r.uniform();
            if (x < a) {
            } else if (x < a + b) {
                v |= 1 << bit;
            } else if (x < a + b + c) {
                u |= 1 << bit;
            } else {
                u |= 1 << bit;
                v |= 1 << bit;
            }
        }
        e.emplace_back(u, v);
    }
    return build_csr(n, e);
}

thread_local Csr g_last;

}  // namespace

extern "C" {

// Generate into an internal buffer; returns n and nnz, then gg_copy() fills
// caller arrays of n+1 offsets and nnz neighbours.
int gg_sbm(std::int32_t blocks, std::int32_t size, double avg_deg, double intra, std::uint64_t seed, std::int32_t* n,
           std::int64_t* nnz) {
    g_last = sbm(blocks, size, avg_deg, intra, seed);
    *n = static_cast<std::int32_t>(g_last.offsets.size()) - 1;
    *nnz = static_cast<std::int64_t>(g_last.nbr.size());
    return 0;
}

int gg_lfr(std::int32_t n_nodes, double avg_deg, double tau1, double kmax, double tau2, double cmin, double cmax,
           double mu, std::uint64_t seed, std::int32_t* n, std::int64_t* nnz) {
    g_last = lfr(n_nodes, avg_deg, tau1, kmax, tau2, cmin, cmax, mu, seed);
    *n = static_cast<std::int32_t>(g_last.offsets.size()) - 1;
    *nnz = static_cast<std::int64_t>(g_last.nbr.size());
    return 0;
}

int gg_rmat(int scale, double edge_factor, double a, double b, double c, std::uint64_t seed, std::int32_t* n,
            std::int64_t* nnz) {
    g_last = rmat(scale, edge_factor, a, b, c, seed);
    *n = static_cast<std::int32_t>(g_last.offsets.size()) - 1;
    *nnz = static_cast<std::int64_t>(g_last.nbr.size());
    return 0;
}

// Uniform random graph in the shape of the reference's oracles::random_graph
// (tests/oracles.hpp:134-154): target round(avg_deg*n/2) distinct edges,
// weights U[0.5, 2) unless unit. Edge list output (u < v), caller sized.
std::int64_t gg_random_edges(std::int32_t n, double avg_deg, int unit, std::uint64_t seed, std::int32_t* u,
                             std::int32_t* v, double* w, std::int64_t cap) {
    Rng r(seed);
    const std::int64_t target = std::max<std::int64_t>(1, static_cast<std::int64_t>(avg_deg * n / 2.0));
    std::vector<std::uint64_t> seen;
    std::int64_t m = 0;
    for (std::int64_t att = 0; m < target && att < 20 * target && m < cap; ++att) {
        std::int32_t a = static_cast<std::int32_t>(r.below(n)), b = static_cast<std::int32_t>(r.below(n));
        if (a == b) continue;
        if (a > b) std::swap(a, b);
        const std::uint64_t key = (static_cast<std::uint64_t>(a) << 32) | static_cast<std::uint32_t>(b);
        if (std::find(seen.begin(), seen.end(), key) != seen.end()) continue;
        seen.push_back(key);
        u[m] = a;
        v[m] = b;
        w[m] = unit ? 1.0 : 0.5 + 1.5 * r.uniform();
        ++m;
    }
    if (m == 0 && cap > 0) {
        u[0] = 0;
        v[0] = n > 1 ? 1 : 0;
        w[0] = 1.0;
        m = 1;
    }
    return m;
}

// Planted community of every node of the last sbm/lfr graph (n entries);
// returns 0 when the last generator has none.
int gg_labels(std::int32_t* out) {
    if (g_labels.empty()) return 0;
    std::memcpy(out, g_labels.data(), g_labels.size() * sizeof(std::int32_t));
    return 1;
}

int gg_copy(std::int64_t* offsets, std::int32_t* nbr) {
    std::memcpy(offsets, g_last.offsets.data(), g_last.offsets.size() * sizeof(std::int64_t));
    std::memcpy(nbr, g_last.nbr.data(), g_last.nbr.size() * sizeof(std::int32_t));
    g_last = Csr{};
    return 0;
}

}  // extern "C"

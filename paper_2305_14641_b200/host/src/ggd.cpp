// Graph Gradient Descent through the C-ABI (reference: src/ggd.cpp:7-62).
#include "graphqc/ggd.hpp"

#include <algorithm>

#include "device.hpp"

namespace graphqc {

namespace {

std::vector<std::int32_t> centers_of(const std::vector<std::int32_t>& center) {  // ggd.cpp:48-50
    std::vector<std::int32_t> out;
    for (std::int32_t i = 0; i < static_cast<std::int32_t>(center.size()); ++i)
        if (center[i] == i) out.push_back(i);
    return out;
}

}  // namespace

SuccessorMap build_successors(const Graph& g, const PotentialField& pf) {
    if (static_cast<std::int32_t>(pf.values.size()) != g.num_nodes())
        throw std::invalid_argument("potential field does not match graph size");
    SuccessorMap s;
    s.succ.resize(g.num_nodes());
    const gqc_csr c = detail::to_gqc(g);
    detail::check(gqc_build_successors(&c, pf.values.data(), s.succ.data()));
    return s;
}

ClusterAssignment resolve_centers(const SuccessorMap& s) {
    const std::int32_t n = static_cast<std::int32_t>(s.succ.size());
    ClusterAssignment out;
    out.center.resize(n);
    out.cluster_index.resize(n);
    detail::check(gqc_resolve_centers(n, s.succ.data(), out.center.data(), out.cluster_index.data(),
                                      &out.num_clusters));
    out.centers = centers_of(out.center);
    return out;
}

std::vector<ClusterAssignment> cluster_batch(const Graph& g, std::span<const double> sigmas, bool with_center) {
    if (sigmas.empty()) return {};
    for (double s : sigmas)
        if (!(s > 0.0)) throw std::invalid_argument("sigma must be positive");
    const std::size_t n = static_cast<std::size_t>(g.num_nodes());
    const gqc_csr c = detail::to_gqc(g);
    std::vector<ClusterAssignment> out(sigmas.size());
    // bounded host staging: 64 sigmas per device call
    constexpr std::size_t kChunk = 64;
    std::vector<std::int32_t> center, ci, k;
    std::vector<std::int64_t> intra;
    const bool unit = c.w == nullptr;  // modularity's intra term comes back exact with the labels
    for (std::size_t q0 = 0; q0 < sigmas.size(); q0 += kChunk) {
        const std::size_t m = std::min(kChunk, sigmas.size() - q0);
        center.resize(with_center ? m * n : 0);
        ci.resize(m * n);
        k.resize(m);
        intra.resize(unit ? m : 0);
        detail::check(gqc_cluster_sweep_intra(&c, sigmas.data() + q0, static_cast<std::int32_t>(m), nullptr, nullptr,
                                              with_center ? center.data() : nullptr, ci.data(), k.data(),
                                              unit ? intra.data() : nullptr));
        for (std::size_t q = 0; q < m; ++q) {
            ClusterAssignment& a = out[q0 + q];
            a.cluster_index.assign(ci.begin() + q * n, ci.begin() + (q + 1) * n);
            a.num_clusters = k[q];
            if (unit) {
                a.intra_weight = static_cast<double>(intra[q]);
                a.intra_labels_hash = labels_hash(a.cluster_index);
            }
            if (with_center) {
                a.center.assign(center.begin() + q * n, center.begin() + (q + 1) * n);
                a.centers = centers_of(a.center);
            }
        }
    }
    return out;
}

std::uint64_t labels_hash(const std::vector<std::int32_t>& labels) {
    std::uint64_t h = 0x9E3779B97F4A7C15ull ^ labels.size();
    for (std::int32_t x : labels) {
        h ^= static_cast<std::uint32_t>(x);
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 29;
    }
    return h;
}

ClusterAssignment cluster(const Graph& g, double sigma, int workers) {  // ggd.cpp:59-62
    if (!(sigma > 0.0)) throw std::invalid_argument("sigma must be positive");
    if (workers < 1) throw std::invalid_argument("workers must be at least 1");
    return std::move(cluster_batch(g, std::span<const double>(&sigma, 1))[0]);
}

}  // namespace graphqc

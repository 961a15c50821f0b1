// Graph Gradient Descent through the C-ABI (reference: src/ggd.cpp:7-62).
#include "graphqc/ggd.hpp"

#include <algorithm>
#include <atomic>

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

namespace {
std::atomic<int> g_max_gpus{0};  // 0: every visible device
}  // namespace

void set_max_gpus(int gpus) {
    if (gpus < 1) throw std::invalid_argument("gpus must be at least 1");
    g_max_gpus = gpus;
}

int max_gpus() {
    const int m = g_max_gpus.load();
    return m > 0 ? m : std::max(1, static_cast<int>(gqc_device_count()));
}

namespace detail {

std::vector<std::int32_t> devices_for(const Graph& g, int workers) {
    // below ~2^22 CSR entries per extra device the per-device upload and
    // context costs more than the rows it takes off the first device
    const long long nnz = 2 * g.num_edges();
    const int by_size = static_cast<int>(std::min<long long>(32, 1 + nnz / (1ll << 22)));
    const int k = std::max(1, std::min({workers, max_gpus(), std::max(1, static_cast<int>(gqc_device_count())),
                                        by_size, 32}));
    std::vector<std::int32_t> d(k);
    for (int r = 0; r < k; ++r) d[r] = r;
    return d;
}

std::vector<ClusterAssignment> cluster_batch_intra(const Graph& g, std::span<const double> sigmas, bool with_center,
                                                   int workers, std::vector<double>* intra_out) {
    if (sigmas.empty()) return {};
    for (double s : sigmas)
        if (!(s > 0.0)) throw std::invalid_argument("sigma must be positive");
    if (workers < 1) throw std::invalid_argument("workers must be at least 1");
    const std::size_t n = static_cast<std::size_t>(g.num_nodes());
    const gqc_csr c = to_gqc(g);
    const std::vector<std::int32_t> dev = devices_for(g, workers);
    std::vector<ClusterAssignment> out(sigmas.size());
    // bounded host staging: 64 sigmas per device call
    constexpr std::size_t kChunk = 64;
    std::vector<std::int32_t> center, ci, k;
    std::vector<std::int64_t> intra;
    const bool unit = c.w == nullptr && intra_out;  // modularity's intra term comes back exact with the labels
    if (intra_out) intra_out->assign(unit ? sigmas.size() : 0, 0.0);
    for (std::size_t q0 = 0; q0 < sigmas.size(); q0 += kChunk) {
        const std::size_t m = std::min(kChunk, sigmas.size() - q0);
        center.resize(with_center ? m * n : 0);
        ci.resize(m * n);
        k.resize(m);
        intra.resize(unit ? m : 0);
        check(gqc_cluster_sweep_multi(&c, sigmas.data() + q0, static_cast<std::int32_t>(m), dev.data(),
                                      static_cast<std::int32_t>(dev.size()), nullptr, nullptr,
                                      with_center ? center.data() : nullptr, ci.data(), k.data(),
                                      unit ? intra.data() : nullptr));
        for (std::size_t q = 0; q < m; ++q) {
            ClusterAssignment& a = out[q0 + q];
            a.cluster_index.assign(ci.begin() + q * n, ci.begin() + (q + 1) * n);
            a.num_clusters = k[q];
            if (unit) (*intra_out)[q0 + q] = static_cast<double>(intra[q]);
            if (with_center) {
                a.center.assign(center.begin() + q * n, center.begin() + (q + 1) * n);
                a.centers = centers_of(a.center);
            }
        }
    }
    return out;
}

}  // namespace detail

std::vector<ClusterAssignment> cluster_batch(const Graph& g, std::span<const double> sigmas, bool with_center,
                                             int workers) {
    return detail::cluster_batch_intra(g, sigmas, with_center, workers, nullptr);
}

ClusterAssignment cluster(const Graph& g, double sigma, int workers) {  // ggd.cpp:59-62
    if (!(sigma > 0.0)) throw std::invalid_argument("sigma must be positive");
    if (workers < 1) throw std::invalid_argument("workers must be at least 1");
    return std::move(cluster_batch(g, std::span<const double>(&sigma, 1), true, workers)[0]);
}

}  // namespace graphqc

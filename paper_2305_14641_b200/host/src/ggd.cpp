// Graph Gradient Descent through the C-ABI (reference: src/ggd.cpp:7-62).
#include "graphqc/ggd.hpp"

#include <algorithm>
#include <atomic>
#include <mutex>
#include <thread>

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

namespace {
// Pinned host staging for label downloads (gqc_host_alloc), kept by the
// process and grown on demand; one user at a time.
struct PinnedStage {
    static std::mutex& mu() {
        static std::mutex m;
        return m;
    }
    static std::pair<void*, std::size_t>& buf() {
        static std::pair<void*, std::size_t> b{nullptr, 0};
        return b;
    }
    std::unique_lock<std::mutex> lock{mu()};
    std::int32_t* get(std::size_t count) {
        auto& [p, cap] = buf();
        const std::size_t bytes = std::max<std::size_t>(count, 1) * sizeof(std::int32_t);
        if (bytes > cap) {
            if (p) gqc_host_free(p);
            p = gqc_host_alloc(bytes);
            if (!p) throw std::bad_alloc();
            cap = bytes;
        }
        return static_cast<std::int32_t*>(p);
    }
};
}  // namespace

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
    // bounded host staging: 64 sigmas per device call, in pinned memory so
    // the label downloads run at PCIe speed under the next GGD chunk; every
    // assignment then copies its slice (in parallel over sigmas)
    constexpr std::size_t kChunk = 64;
    std::vector<std::int32_t> k;
    std::vector<std::int64_t> intra;
    const bool unit = c.w == nullptr && intra_out;  // modularity's intra term comes back exact with the labels
    if (intra_out) intra_out->assign(unit ? sigmas.size() : 0, 0.0);
    PinnedStage stage;
    for (std::size_t q0 = 0; q0 < sigmas.size(); q0 += kChunk) {
        const std::size_t m = std::min(kChunk, sigmas.size() - q0);
        std::int32_t* ci = stage.get(m * n * (with_center ? 2 : 1));
        std::int32_t* center = with_center ? ci + m * n : nullptr;
        k.resize(m);
        intra.resize(unit ? m : 0);
        check(gqc_cluster_sweep_multi(&c, sigmas.data() + q0, static_cast<std::int32_t>(m), dev.data(),
                                      static_cast<std::int32_t>(dev.size()), nullptr, nullptr, center, ci, k.data(),
                                      unit ? intra.data() : nullptr));
        const unsigned T = std::max(1u, std::min<unsigned>(static_cast<unsigned>(m),
                                                          n < 50000 ? 1u : std::thread::hardware_concurrency()));
        auto fill = [&](std::size_t qa, std::size_t qb) {
            for (std::size_t q = qa; q < qb; ++q) {
                ClusterAssignment& a = out[q0 + q];
                a.cluster_index.assign(ci + q * n, ci + (q + 1) * n);
                a.num_clusters = k[q];
                if (unit) (*intra_out)[q0 + q] = static_cast<double>(intra[q]);
                if (with_center) {
                    a.center.assign(center + q * n, center + (q + 1) * n);
                    a.centers = centers_of(a.center);
                }
            }
        };
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < T; ++t) pool.emplace_back(fill, m * t / T, m * (t + 1) / T);
        fill(0, m / T);
        for (std::thread& th : pool) th.join();
    }
    return out;
}

}  // namespace detail

void reserve_for(const Graph& g, int n_sigma, bool with_center) {
    if (n_sigma < 1) throw std::invalid_argument("sigma count must be at least 1");
    const int m = std::min(n_sigma, 64);  // cluster_batch_intra's chunk
    const std::size_t n = static_cast<std::size_t>(g.num_nodes());
    detail::check(gqc_reserve(g.num_nodes(), 2 * g.num_edges(), m));
    detail::PinnedStage stage;
    (void)stage.get(static_cast<std::size_t>(m) * n * (with_center ? 2 : 1));
}

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

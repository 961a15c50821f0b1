// Potential field through the C-ABI (reference: src/potential.cpp:39-87).
#include "graphqc/potential.hpp"

#include "device.hpp"
#include "graphqc/ggd.hpp"

namespace graphqc {

namespace {

void check_sigma(double sigma) {  // potential.cpp:39-42
    if (!(sigma > 0.0)) throw std::invalid_argument("sigma must be positive");
}

}  // namespace

double node_potential(const Graph& g, std::int32_t node, double sigma) {
    check_sigma(sigma);
    g.check_node(node);
    const gqc_csr c = detail::to_gqc(g);
    double v = 0.0;
    detail::check(gqc_node_potential(&c, node, sigma, &v));
    return v;
}

PotentialField compute_potentials(const Graph& g, double sigma) {
    check_sigma(sigma);
    PotentialField pf{sigma, g.default_distance(), std::vector<double>(g.num_nodes())};
    const gqc_csr c = detail::to_gqc(g);
    detail::check(gqc_potentials(&c, &sigma, 1, pf.values.data()));
    return pf;
}

// potential.cpp:62-87: rows in contiguous blocks over `workers` workers —
// here GPUs (detail::devices_for), each block's rows on its own device.
PotentialField compute_potentials_parallel(const Graph& g, double sigma, int workers) {
    check_sigma(sigma);
    if (workers < 1) throw std::invalid_argument("workers must be at least 1");
    PotentialField pf{sigma, g.default_distance(), std::vector<double>(g.num_nodes())};
    const gqc_csr c = detail::to_gqc(g);
    const std::vector<std::int32_t> dev = detail::devices_for(g, workers);
    detail::check(gqc_potentials_multi(&c, &sigma, 1, dev.data(), static_cast<std::int32_t>(dev.size()),
                                       pf.values.data()));
    return pf;
}

std::vector<PotentialField> compute_potentials_batch(const Graph& g, std::span<const double> sigmas) {
    if (sigmas.empty()) return {};
    for (double s : sigmas) check_sigma(s);
    const std::size_t n = static_cast<std::size_t>(g.num_nodes());
    std::vector<double> all(n * sigmas.size());
    const gqc_csr c = detail::to_gqc(g);
    detail::check(gqc_potentials(&c, sigmas.data(), static_cast<std::int32_t>(sigmas.size()), all.data()));
    std::vector<PotentialField> out(sigmas.size());
    for (std::size_t q = 0; q < sigmas.size(); ++q)
        out[q] = PotentialField{sigmas[q], g.default_distance(),
                                std::vector<double>(all.begin() + q * n, all.begin() + (q + 1) * n)};
    return out;
}

}  // namespace graphqc

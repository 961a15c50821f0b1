// graphqc-compatible host facade: Graph Gradient Descent (reference:
// include/graphqc/ggd.hpp:15-37), on the GPU through the C-ABI.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <vector>

#include "graphqc/graph.hpp"
#include "graphqc/potential.hpp"

namespace graphqc {

struct SuccessorMap {
    std::vector<std::int32_t> succ;
};

struct ClusterAssignment {
    std::vector<std::int32_t> center;
    std::vector<std::int32_t> cluster_index;
    std::vector<std::int32_t> centers;
    std::int32_t num_clusters = 0;
    // Extension (not in the reference struct): modularity's intra-cluster
    // weight of a unit-weight graph, counted on the device by cluster_batch
    // (exact); modularity() then skips its O(nnz) row loop — only while
    // cluster_index still hashes to intra_labels_hash (edited labels fall
    // back to the full loop).
    std::optional<double> intra_weight;
    std::uint64_t intra_labels_hash = 0;
};

// Hash of a labelling that guards ClusterAssignment::intra_weight.
std::uint64_t labels_hash(const std::vector<std::int32_t>& labels);

SuccessorMap build_successors(const Graph& g, const PotentialField& pf);
ClusterAssignment resolve_centers(const SuccessorMap& s);
ClusterAssignment cluster(const Graph& g, double sigma, int workers = 1);
// One assignment per sigma from one batched device sweep. with_center = false
// fills only cluster_index / num_clusters (all a sweep's metrics need).
std::vector<ClusterAssignment> cluster_batch(const Graph& g, std::span<const double> sigmas, bool with_center = true);

}  // namespace graphqc

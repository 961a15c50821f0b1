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
};

SuccessorMap build_successors(const Graph& g, const PotentialField& pf);
ClusterAssignment resolve_centers(const SuccessorMap& s);
// `workers` (>= 1, as the reference validates) is the number of GPUs the rows
// are sharded over: min(workers, max_gpus(), visible devices), one GPU for
// graphs too small to gain from more (same bits for any count).
ClusterAssignment cluster(const Graph& g, double sigma, int workers = 1);
// One assignment per sigma from one batched device sweep over `workers` GPUs
// (as cluster). with_center = false fills only cluster_index / num_clusters
// (all a sweep's metrics need).
std::vector<ClusterAssignment> cluster_batch(const Graph& g, std::span<const double> sigmas, bool with_center = true,
                                             int workers = 1);

// Upper bound on the GPUs a call shards over (default: every visible device;
// the CLI's --gpus). Not a reference function: the reference's `workers` are
// host threads.
void set_max_gpus(int gpus);
int max_gpus();

// Optional, not a reference function: sizes the device buffers and the
// pinned label staging for cluster / cluster_batch calls on g with up to
// n_sigma sigmas (gqc_reserve), so the first call of a process does not
// allocate on its critical path. The CLI runs it on its warm-up thread.
void reserve_for(const Graph& g, int n_sigma, bool with_center);

namespace detail {
// cluster_batch plus modularity's intra-cluster weight per sigma, counted
// exactly on the device with the labels (unit-weight graphs; empty
// otherwise). Used by run_sweep only, for the assignments it just made.
std::vector<ClusterAssignment> cluster_batch_intra(const Graph& g, std::span<const double> sigmas, bool with_center,
                                                   int workers, std::vector<double>* intra);
// The device list of a call with `workers` workers on g.
std::vector<std::int32_t> devices_for(const Graph& g, int workers);
}  // namespace detail

}  // namespace graphqc

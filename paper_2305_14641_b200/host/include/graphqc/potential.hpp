// graphqc-compatible host facade: potential field (reference:
// include/graphqc/potential.hpp:22-37). Computed on the GPU through the C-ABI
// (include/gqc.h); values are bit-identical to the reference's ascending-j sums.
// The reference stores values in an Eigen::VectorXd; here a std::vector<double>
// with the same .size(), operator[] and == semantics.
#pragma once

#include <cstdint>
#include <vector>

#include "graphqc/graph.hpp"

namespace graphqc {

struct PotentialField {
    double sigma = 1.0;
    double default_distance = 10.0;
    std::vector<double> values;
};

double node_potential(const Graph& g, std::int32_t node, double sigma);
PotentialField compute_potentials(const Graph& g, double sigma);
// `workers` (>= 1, validated like the reference) = GPUs the rows are sharded over
// (see cluster in ggd.hpp); the field is the same bits for any count.
PotentialField compute_potentials_parallel(const Graph& g, double sigma, int workers);
// Batched: one field per sigma from one device pass over the CSR.
std::vector<PotentialField> compute_potentials_batch(const Graph& g, std::span<const double> sigmas);

}  // namespace graphqc

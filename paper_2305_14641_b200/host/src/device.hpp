// Facade <-> C-ABI glue: CSR view and status -> exception mapping.
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "../../../include/gqc.h"
#include "graphqc/graph.hpp"

namespace graphqc::detail {

inline gqc_csr to_gqc(const Graph& g) {
    const Graph::CsrView v = g.csr();
    return gqc_csr{g.num_nodes(), 2 * g.num_edges(), v.offsets, v.nbr, v.unit ? nullptr : v.weights,
                   g.default_distance()};
}

// The C-ABI's status codes mirror the reference's exception classes.
inline void check(gqc_status st) {
    if (st == GQC_OK) return;
    const std::string msg = gqc_last_error();
    switch (st) {
        case GQC_EINVAL: throw std::invalid_argument(msg);
        case GQC_ERANGE: throw std::out_of_range(msg);
        case GQC_ECYCLE: throw std::logic_error(msg);
        case GQC_EIO: throw IoError(msg);
        case GQC_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error("device failure: " + msg);
    }
}

}  // namespace graphqc::detail

// Host exp provider and per-sigma constant tables.
//
// The reference evaluates gauss = exp(-inv * dist2) at potential.cpp:26 with
// Eigen's ArrayXd::exp. In the default Release build (no -march) that is
// Eigen 3.4's pexp_double on SSE2 Packet2d for every whole packet, and scalar
// std::exp (glibc) for the last element when N is odd. Bit parity of the
// potentials therefore needs the exact exp bits, so exp never runs in a
// "close enough" device intrinsic: it runs here, on the host, with the same
// arithmetic the reference's build performs, and the device kernels only see
// the resulting constants. (Weighted graphs additionally use a device port of
// the same pexp, gqc_pexp_dev in kernels.cu, which performs the identical
// sequence of IEEE-rounded operations.)
//
// Compiled with -O2 -ffp-contract=off and no -march: scalar SSE2 double, no
// FMA, i.e. the same roundings as one SSE2 lane of the reference.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "gqc_internal.h"

namespace gqc {

static double pow2_bits(std::int32_t k) {
    const std::uint64_t bits = static_cast<std::uint64_t>(static_cast<std::int64_t>(k) + 1023) << 52;
    double d;
    std::memcpy(&d, &bits, sizeof d);
    return d;
}

// Eigen 3.4 pexp_double, one lane (GenericPacketMathFunctions.h), with
// pldexp<Packet2d> from SSE/PacketMath.h (2^e split into four factors).
double host_pexp(double x0) {
    double x = std::max(std::min(x0, 709.784), -709.784);
    double fx = std::floor(1.4426950408889634073599 * x + 0.5);
    x = x - fx * 0.693145751953125;
    x = x - fx * 1.42860682030941723212e-6;
    const double x2 = x * x;
    double px = (1.26177193074810590878e-4 * x2 + 3.02994407707441961300e-2) * x2 + 9.99999999999999999910e-1;
    px = px * x;
    double qx = ((3.00198505138664455042e-6 * x2 + 2.52448340349684104192e-3) * x2 + 2.27265548208155028766e-1) * x2 +
                2.00000000000000000009e0;
    double r = px / (qx - px);
    r = 2.0 * r + 1.0;
    const double e = std::min(std::max(fx, -2099.0), 2099.0);
    const std::int32_t ei = static_cast<std::int32_t>(e);
    std::int32_t b = ei >> 2;
    const double c = pow2_bits(b);
    double out = r * c * c * c;
    out = out * pow2_bits(ei - 3 * b);
    return out > x0 ? out : x0;
}

double host_glibc_exp(double x) { return std::exp(x); }

// potential.cpp:39-42 (order: 2.0*sigma, then *sigma, then 1.0/...)
double inv_two_sigma_sq(double sigma) { return 1.0 / (2.0 * sigma * sigma); }

// Per-sigma constants for unit-weight neighbours and non-adjacent pairs.
// For column j the reference computes d2[j] * exp((-inv) * d2[j]).
SigmaConsts make_sigma_consts(double sigma, double W, int exp_mode) {
    SigmaConsts c{};
    const double inv = inv_two_sigma_sq(sigma);
    const double neg = -inv;
    const double w2 = W * W;  // potential.cpp:19
    const double aW = neg * w2;
    const double a1 = neg * 1.0;
    auto body_exp = [&](double a) { return exp_mode == 0 ? host_pexp(a) : host_glibc_exp(a); };
    c.inv = inv;
    c.neg_inv = neg;
    c.eW = body_exp(aW);
    c.pW = w2 * c.eW;
    c.e1 = body_exp(a1);
    c.p1 = 1.0 * c.e1;
    // N-odd tail column (Eigen's scalar remainder): glibc std::exp.
    c.eWt = host_glibc_exp(aW);
    c.pWt = w2 * c.eWt;
    c.e1t = host_glibc_exp(a1);
    c.p1t = 1.0 * c.e1t;
    return c;
}

// k-hop extension: the hop-h term of the reference loop with dist2 = h*h
// (potential.cpp:26, :32-33 with d = h): e = exp((-inv) * d2), p = d2 * e.
void fill_khop_table(KhopTable& t, int s, double sigma, int hop_cap, int exp_mode) {
    const double neg = -inv_two_sigma_sq(sigma);
    for (int h = 0; h <= kMaxHopCap; ++h) {
        const double d = static_cast<double>(h);
        const double d2 = d * d;
        const double a = neg * d2;
        const bool used = h >= 1 && h <= hop_cap;
        t.e[h][s] = used ? (exp_mode == 0 ? host_pexp(a) : host_glibc_exp(a)) : 0.0;
        t.p[h][s] = d2 * t.e[h][s];
        t.et[h][s] = used ? host_glibc_exp(a) : 0.0;
        t.pt[h][s] = d2 * t.et[h][s];
    }
}

}  // namespace gqc

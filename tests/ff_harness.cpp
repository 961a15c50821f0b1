// CPU harness for the exact fast-forward (paper_2305_14641_b200/csrc/ff_chain.cuh):
// the same source the sm_100a kernel compiles, checked against naive
// sequential adds on randomized cases (binade crossings, half-ulp ties,
// subnormals, fixed points) and on row-like sequences of runs and terms.
// Built by tests/test_ff_cpu.py with g++ -O2 -ffp-contract=off (no -march).
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <cmath>
#include <vector>

static thread_local long long g_walk_iters = 0;
#define GQC_WALK_COUNT() (++g_walk_iters)
#include "ff_chain.cuh"

using namespace gqc::ffc;

namespace {

struct Rng {
    std::uint64_t s;
    std::uint64_t next() {
        std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uni() { return (next() >> 11) * 0x1.0p-53; }
    int below(int n) { return static_cast<int>(uni() * n); }
};

double from_bits(std::uint64_t b) {
    double d;
    std::memcpy(&d, &b, sizeof d);
    return d;
}

// A positive double with a random biased exponent in [elo, ehi] (0 = subnormal)
// and a mantissa with a random number of trailing zero bits (ties).
double rand_double(Rng& r, int elo, int ehi) {
    const int e = elo + r.below(ehi - elo + 1);
    std::uint64_t mant = r.next() & ((1ull << 52) - 1);
    const int tz = r.below(4) == 0 ? r.below(53) : 0;
    if (tz > 0) mant &= ~((1ull << tz) - 1);
    if (e == 0 && mant == 0) mant = 1;
    return from_bits((static_cast<std::uint64_t>(e) << 52) | mant);
}

double naive(double s, double c, long long L) {
    for (long long t = 0; t < L; ++t) s = s + c;
    return s;
}

int rand_len(Rng& r, int maxL) {
    // log-uniform in [1, maxL]
    const double x = r.uni() * __builtin_log(static_cast<double>(maxL));
    int L = static_cast<int>(__builtin_exp(x));
    return L < 1 ? 1 : (L > maxL ? maxL : L);
}

}  // namespace

extern "C" {

// Single runs from arbitrary (s, c, L). Returns the number of mismatches;
// the first one is written to bad[0..2] = (s, c, L).
long long fft_single(std::uint64_t seed, int ncases, int maxL, double* bad) {
    Rng r{seed};
    long long mism = 0;
    for (int k = 0; k < ncases; ++k) {
        const int mode = r.below(5);
        double c, s;
        if (mode == 0) {  // subnormal / tiny regime
            c = rand_double(r, 0, 3);
            s = r.below(3) == 0 ? 0.0 : rand_double(r, 0, 6);
        } else {
            const int ec = 1 + r.below(1100);
            c = rand_double(r, ec > 2000 ? 2000 : ec, ec > 2000 ? 2000 : ec);
            const int es = ec + r.below(70) - 8;
            s = (mode == 1 || es < 0) ? 0.0 : rand_double(r, es < 0 ? 0 : es, es < 0 ? 0 : (es > 2000 ? 2000 : es));
        }
        const int L = rand_len(r, maxL);
        Chain ch = make_chain(s, c);
        ff_run(ch, c, L);
        const double ref = naive(s, c, L);
        if (std::memcmp(&ch.s, &ref, sizeof ref) != 0) {
            if (mism == 0 && bad) {
                bad[0] = s;
                bad[1] = c;
                bad[2] = L;
            }
            ++mism;
        }
    }
    return mism;
}

// Row-like sequences: a chain with a fixed W constant receives runs of W
// terms interleaved with single larger terms (neighbours) and a +1 (self),
// the cache persisting across runs exactly as in the kernel.
long long fft_rows(std::uint64_t seed, int nrows, int ncols, double* bad) {
    Rng r{seed};
    long long mism = 0;
    for (int row = 0; row < nrows; ++row) {
        const int ew = 1 + r.below(1060);
        const double c = rand_double(r, ew, ew);
        const double term = rand_double(r, ew + r.below(40), ew + 40);
        const int deg = 1 + r.below(40);
        Chain ch = make_chain(0.0, c);
        double ref = 0.0;
        int pos = 0;
        const int self = r.below(ncols);
        for (int q = 0; q <= deg; ++q) {
            const int col = q == deg ? ncols : pos + r.below((ncols - pos) / (deg - q + 1) * 2 + 1);
            const int stop = col > ncols ? ncols : col;
            const int L = stop - pos;
            if (L > 0) {
                ff_run(ch, c, L);
                ref = naive(ref, c, L);
            }
            if (stop >= ncols) break;
            const double t = (stop == self) ? 1.0 : term;
            ch.s = ch.s + t;
            ref = ref + t;
            pos = stop + 1;
        }
        if (std::memcmp(&ch.s, &ref, sizeof ref) != 0) {
            if (mism == 0 && bad) {
                bad[0] = c;
                bad[1] = term;
                bad[2] = row;
            }
            ++mism;
        }
    }
    return mism;
}


// Prefix segments: P(L) for every L < n against the naive trajectory.
long long fft_prefix(std::uint64_t seed, int ncases, int maxn, double* bad) {
    Rng r{seed};
    long long mism = 0;
    int t[kPrefixCap];
    double s0[kPrefixCap], inc[kPrefixCap];
    for (int k = 0; k < ncases; ++k) {
        const int ec = r.below(8) == 0 ? r.below(4) : 1 + r.below(1100);
        const double c = rand_double(r, ec, ec);
        const int n = 1 + rand_len(r, maxn);
        int count = 0, t_end = 0;
        double s_end = 0.0;
        build_prefix(c, n, t, s0, inc, &count, &t_end, &s_end);
        double ref = 0.0;
        for (int L = 0; L < n; ++L) {
            double got;
            if (L < t_end) {
                got = prefix_value(t, s0, inc, count, L);
            } else {
                Chain ch = make_chain(s_end, c);
                ff_run(ch, c, L - t_end);
                got = ch.s;
            }
            if (std::memcmp(&got, &ref, sizeof ref) != 0) {
                if (mism == 0 && bad) {
                    bad[0] = c;
                    bad[1] = n;
                    bad[2] = L;
                }
                ++mism;
                break;
            }
            ref = ref + c;
        }
    }
    return mism;
}

// Two chains (num with p = W^2 e, den with e) through ff_run2, first run via
// the prefix table, exactly as the kernel walks a row.
long long fft_rows2(std::uint64_t seed, int nrows, int ncols, double* bad) {
    Rng r{seed};
    long long mism = 0;
    int tp[2][kPrefixCap];
    double sp[2][kPrefixCap], ip[2][kPrefixCap];
    for (int row = 0; row < nrows; ++row) {
        const int ew = 1 + r.below(1060);
        const double e = rand_double(r, ew, ew);
        const double p = 100.0 * e;
        const double te = rand_double(r, ew + r.below(40), ew + 40);
        const double tpv = 1.0 * te;
        int cnt[2], tend[2];
        double send[2];
        build_prefix(p, ncols, tp[0], sp[0], ip[0], &cnt[0], &tend[0], &send[0]);
        build_prefix(e, ncols, tp[1], sp[1], ip[1], &cnt[1], &tend[1], &send[1]);
        const int deg = 1 + r.below(40);
        const int self = r.below(ncols);
        Chain num = make_chain(0.0, p), den = make_chain(0.0, e);
        double rn = 0.0, rd = 0.0;
        int pos = 0;
        bool first = true;
        for (int q = 0; q <= deg; ++q) {
            int col = q == deg ? ncols : pos + r.below((ncols - pos) / (deg - q + 1) * 2 + 1);
            if (col > ncols) col = ncols;
            const int L = col - pos;
            if (L > 0) {
                if (first) {
                    if (L < tend[0]) num.s = prefix_value(tp[0], sp[0], ip[0], cnt[0], L);
                    else { num.s = send[0]; ff_run(num, p, L - tend[0]); }
                    if (L < tend[1]) den.s = prefix_value(tp[1], sp[1], ip[1], cnt[1], L);
                    else { den.s = send[1]; ff_run(den, e, L - tend[1]); }
                    num.top = 0.0;
                    den.top = 0.0;
                } else {
                    ff_run2(num, p, den, e, L);
                }
                rn = naive(rn, p, L);
                rd = naive(rd, e, L);
            }
            first = false;
            if (col >= ncols) break;
            if (col == self) {
                den.s = den.s + 1.0;
                rd = rd + 1.0;
            } else {
                num.s = num.s + tpv;
                den.s = den.s + te;
                rn = rn + tpv;
                rd = rd + te;
            }
            pos = col + 1;
        }
        if (std::memcmp(&num.s, &rn, sizeof rn) != 0 || std::memcmp(&den.s, &rd, sizeof rd) != 0) {
            if (mism == 0 && bad) {
                bad[0] = e;
                bad[1] = te;
                bad[2] = row;
            }
            ++mism;
        }
    }
    return mism;
}

// fft_rows2 with the single-loop two-chain walk (ff_walk2).
long long fft_rows2w(std::uint64_t seed, int nrows, int ncols, double* bad) {
    Rng r{seed};
    long long mism = 0;
    int tp[2][kPrefixCap];
    double sp[2][kPrefixCap], ip[2][kPrefixCap];
    for (int row = 0; row < nrows; ++row) {
        const int ew = 1 + r.below(1060);
        const double e = rand_double(r, ew, ew);
        const double p = 100.0 * e;
        const double te = rand_double(r, ew + r.below(40), ew + 40);
        const double tpv = 1.0 * te;
        int cnt[2], tend[2];
        double send[2];
        build_prefix(p, ncols, tp[0], sp[0], ip[0], &cnt[0], &tend[0], &send[0]);
        build_prefix(e, ncols, tp[1], sp[1], ip[1], &cnt[1], &tend[1], &send[1]);
        const int deg = 1 + r.below(40);
        const int self = r.below(ncols);
        Chain num = make_chain(0.0, p), den = make_chain(0.0, e);
        double rn = 0.0, rd = 0.0;
        int pos = 0;
        bool first = true;
        for (int q = 0; q <= deg; ++q) {
            int col = q == deg ? ncols : pos + r.below((ncols - pos) / (deg - q + 1) * 2 + 1);
            if (col > ncols) col = ncols;
            const int L = col - pos;
            if (L > 0) {
                if (first) {
                    if (L < tend[0]) num.s = prefix_value(tp[0], sp[0], ip[0], cnt[0], L);
                    else { num.s = send[0]; ff_run(num, p, L - tend[0]); }
                    if (L < tend[1]) den.s = prefix_value(tp[1], sp[1], ip[1], cnt[1], L);
                    else { den.s = send[1]; ff_run(den, e, L - tend[1]); }
                    num.top = 0.0;
                    den.top = 0.0;
                } else {
                    ff_walk2(num, p, den, e, L);
                }
                rn = naive(rn, p, L);
                rd = naive(rd, e, L);
            }
            first = false;
            if (col >= ncols) break;
            if (col == self) {
                den.s = den.s + 1.0;
                rd = rd + 1.0;
            } else {
                num.s = num.s + tpv;
                den.s = den.s + te;
                rn = rn + tpv;
                rd = rd + te;
            }
            pos = col + 1;
        }
        if (std::memcmp(&num.s, &rn, sizeof rn) != 0 || std::memcmp(&den.s, &rd, sizeof rd) != 0) {
            if (mism == 0 && bad) {
                bad[0] = e;
                bad[1] = te;
                bad[2] = row;
            }
            ++mism;
        }
    }
    return mism;
}

double fft_run(double s, double c, int L) {
    Chain ch = make_chain(s, c);
    ff_run(ch, c, L);
    return ch.s;
}

double fft_naive(double s, double c, long long L) { return naive(s, c, L); }


// One accumulator of a unit-weight row through walk_events (neighbours before
// the row's own column, the self term, neighbours after it, the final run),
// as the batched kernel walks it.
static double walk_row(double c, double c1, double cself, const int* nb, int deg, int self, int ncols) {
    struct Cols {
        const int* p;
        int operator()(int q) const { return p[q]; }
    } col{nb};
    const int tc = tie_binade(c), tc1 = tie_binade(c1);
    int k1 = 0;
    while (k1 < deg && nb[k1] < self) ++k1;
    double s = walk_events(0.0, c, c1, tc, tc1, col, 0, k1, 0);
    int pos = k1 ? nb[k1 - 1] + 1 : 0;
    Chain ch = make_chain(s, c);
    ff_run(ch, c, self - pos);
    s = ch.s + cself;
    s = walk_events(s, c, c1, tc, tc1, col, k1, deg, self + 1);
    pos = deg > k1 ? nb[deg - 1] + 1 : self + 1;
    ch = make_chain(s, c);
    ff_run(ch, c, ncols - pos);
    return ch.s;
}

static double naive_row(double c, double c1, double cself, const int* nb, int deg, int self, int ncols) {
    double s = 0.0;
    int k = 0;
    for (int j = 0; j < ncols; ++j) {
        if (j == self) s = s + cself;
        else if (k < deg && nb[k] == j) s = s + c1, ++k;
        else s = s + c;
    }
    return s;
}

// Random rows (degree, neighbour columns, self), random constants with tie-prone
// mantissas plus the QC constants of random sigmas; both accumulators. Returns
// mismatches; bad = (c, c1, row). iters_out (optional) = walk iterations.
long long fft_walk(std::uint64_t seed, int nrows, int ncols, double* bad, long long* iters_out) {
    Rng r{seed};
    long long mism = 0;
    std::vector<int> nb;
    g_walk_iters = 0;
    for (int row = 0; row < nrows; ++row) {
        const int deg = r.below(4) == 0 ? r.below(400) : r.below(40);
        const int self = r.below(ncols);
        nb.clear();
        for (int q = 0; q < deg; ++q) {
            const int j = r.below(ncols);
            if (j != self) nb.push_back(j);
        }
        std::sort(nb.begin(), nb.end());
        nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
        double c, c1;
        if (r.below(2)) {
            const double sigma = 0.05 + 40.0 * r.uni();
            const double inv = 1.0 / (2.0 * sigma * sigma);
            c = std::exp(-inv * 100.0);
            c1 = std::exp(-inv);
            if (r.below(2)) c = 100.0 * c, c1 = 1.0 * c1;  // numerator constants
        } else {
            const int ec = 1 + r.below(1060);
            c = rand_double(r, ec, ec);
            c1 = rand_double(r, ec + r.below(45), ec + 45);
            if (r.below(8) == 0) c1 = c;
        }
        const double cself = r.below(2) ? 1.0 : 0.0;
        const double got = walk_row(c, c1, cself, nb.data(), static_cast<int>(nb.size()), self, ncols);
        const double ref = naive_row(c, c1, cself, nb.data(), static_cast<int>(nb.size()), self, ncols);
        if (std::memcmp(&got, &ref, sizeof ref) != 0) {
            if (mism == 0 && bad) {
                bad[0] = c;
                bad[1] = c1;
                bad[2] = row;
            }
            ++mism;
        }
    }
    if (iters_out) *iters_out = g_walk_iters;
    return mism;
}

}  // extern "C"

extern "C" long long fft_walk_row_iters(double c, double c1, double cself, const int* nb, int deg, int self,
                                        int ncols, double* out) {
    g_walk_iters = 0;
    *out = walk_row(c, c1, cself, nb, deg, self, ncols);
    return g_walk_iters;
}

// Multi-class batched walk (walk_events_multi, the k-hop extension): rows of
// W runs, events of NC = 2 or 3 classes with their own constants, the self
// term, walked in chunks of 32 events split at the self column like the
// kernel, against naive sequential adds. Returns mismatches.
namespace {
template <int NC>
struct ChunkEv {
    const int* cols;
    const int* kls;
    int cnt_tab[33][NC];  // cnt_tab[q + 1][k] = class-k events among [0, q]
    int col(int q) const { return cols[q]; }
    int cls(int q) const { return kls[q]; }
    int cnt(int q, int k) const { return cnt_tab[q + 1][k]; }
};

template <int NC>
double walk_row_multi(double c, const double* cc, double cself, const int* nb, const int* kl, int deg, int self,
                      int ncols) {
    int tie[NC];
    for (int k = 0; k < NC; ++k) tie[k] = tie_binade(cc[k]);
    const int tc = tie_binade(c);
    double s = 0.0;
    int pos = 0;
    bool self_pending = true;
    for (int b = 0; b < deg; b += 32) {
        const int n = std::min(32, deg - b);
        ChunkEv<NC> ev{nb + b, kl + b, {}};
        for (int q = 0; q < n; ++q)
            for (int k = 0; k < NC; ++k) ev.cnt_tab[q + 1][k] = ev.cnt_tab[q][k] + (kl[b + q] == k);
        int j = 0;
        while (j < n) {
            int r = n;
            if (self_pending) {
                r = j;
                while (r < n && nb[b + r] < self) ++r;
            }
            if (r > j) {
                s = walk_events_multi<NC>(s, c, tc, cc, tie, ev, j, r, pos);
                pos = nb[b + r - 1] + 1;
                j = r;
            }
            if (self_pending && j < n) {
                Chain ch = make_chain(s, c);
                ff_run(ch, c, self - pos);
                s = ch.s + cself;
                pos = self + 1;
                self_pending = false;
            }
        }
    }
    Chain ch = make_chain(s, c);
    if (self_pending) {
        ff_run(ch, c, self - pos);
        ch.s = ch.s + cself;
        pos = self + 1;
        ch.top = 0.0;
    }
    ff_run(ch, c, ncols - pos);
    return ch.s;
}

double naive_row_multi(double c, const double* cc, double cself, const int* nb, const int* kl, int deg, int self,
                       int ncols) {
    double s = 0.0;
    int k = 0;
    for (int j = 0; j < ncols; ++j) {
        if (j == self) s = s + cself;
        else if (k < deg && nb[k] == j) s = s + cc[kl[k]], ++k;
        else s = s + c;
    }
    return s;
}
}  // namespace

extern "C" long long fft_walk_multi(std::uint64_t seed, int nrows, int ncols, int nc, double* bad) {
    Rng r{seed};
    long long mism = 0;
    std::vector<int> nb, kl;
    for (int row = 0; row < nrows; ++row) {
        const int deg = r.below(3) == 0 ? r.below(3000) : r.below(300);
        const int self = r.below(ncols);
        nb.clear();
        for (int q = 0; q < deg; ++q) {
            const int j = r.below(ncols);
            if (j != self) nb.push_back(j);
        }
        std::sort(nb.begin(), nb.end());
        nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
        kl.resize(nb.size());
        for (auto& x : kl) x = r.below(nc);
        double c, cc[3];
        if (r.below(2)) {  // QC constants of a random sigma: W term, hop 1..nc terms (num or den)
            const double sigma = 0.05 + 40.0 * r.uni();
            const double inv = 1.0 / (2.0 * sigma * sigma);
            const bool numer = r.below(2);
            c = std::exp(-inv * 100.0) * (numer ? 100.0 : 1.0);
            for (int k = 0; k < 3; ++k) {
                const double d2 = static_cast<double>((k + 1) * (k + 1));
                cc[k] = std::exp(-inv * d2) * (numer ? d2 : 1.0);
            }
        } else {
            const int ec = 1 + r.below(1060);
            c = rand_double(r, ec, ec);
            for (int k = 0; k < 3; ++k) cc[k] = rand_double(r, ec + r.below(45), ec + 45);
            if (r.below(8) == 0) cc[0] = c;
            if (r.below(8) == 0) cc[1] = cc[0];
        }
        const double cself = r.below(2) ? 1.0 : 0.0;
        const int d = static_cast<int>(nb.size());
        const double got = nc == 2 ? walk_row_multi<2>(c, cc, cself, nb.data(), kl.data(), d, self, ncols)
                                   : walk_row_multi<3>(c, cc, cself, nb.data(), kl.data(), d, self, ncols);
        const double ref = naive_row_multi(c, cc, cself, nb.data(), kl.data(), d, self, ncols);
        if (std::memcmp(&got, &ref, sizeof ref) != 0) {
            if (mism == 0 && bad) {
                bad[0] = c;
                bad[1] = cc[0];
                bad[2] = row;
            }
            ++mism;
        }
    }
    return mism;
}

// Exact fast-forward of sequential fp64 adds (the heart of the FASTFWD
// potential kernel). Host/device portable so the algorithm is unit-tested on
// the CPU against naive sequential adds (tests/test_ff_cpu.py) with the same
// source the sm_100a kernel compiles. Host builds must use -ffp-contract=off.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define GQC_HD __host__ __device__
#else
#define GQC_HD
#endif

// GQC_STEP_FINISH=1: ff_step also finishes a run inside the new binade after
// a settled crossing. Measured: LFR potentials 4.49 -> 4.44 ms but R-MAT
// 10.51 -> 10.90 ms (register pressure in the batched kernel), so off.
#ifndef GQC_STEP_FINISH
#define GQC_STEP_FINISH 0
#endif
// GQC_INCR_REFRESH=1: ff_walk2 moves a stale binade cache up incrementally
// after a crossing neighbour add (refresh_after_add)
#ifndef GQC_INCR_REFRESH
#define GQC_INCR_REFRESH 0
#endif

namespace gqc {
namespace ffc {

#if defined(__CUDA_ARCH__)
__device__ __forceinline__ double gqc_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double gqc_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double gqc_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double gqc_div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double gqc_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
// ~1/a for normal a: MUFU approximation + one Newton step (relative error
// ~2^-44; the jump count it feeds is corrected exactly, see max_steps).
__device__ __forceinline__ double gqc_rcp(double a) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    const double e = __fma_rn(-a, r, 1.0);
    return __fma_rn(r, e, r);
}
__device__ __forceinline__ double gqc_floor(double a) { return floor(a); }
__device__ __forceinline__ long long gqc_bits(double a) { return __double_as_longlong(a); }
__device__ __forceinline__ int gqc_ffsll(long long a) { return __ffsll(a); }
__device__ __forceinline__ int gqc_max(int a, int b) { return max(a, b); }
__device__ __forceinline__ bool gqc_lo_odd(double a) { return __double2loint(a) & 1; }
__device__ __forceinline__ int exp_field(double x) { return (__double2hiint(x) >> 20) & 0x7ff; }
// 2^(f - 1023) for a biased exponent f in [1, 2046]
__device__ __forceinline__ double pow2_field(int f) { return __hiloint2double(f << 20, 0); }
#else
inline double gqc_add(double a, double b) { return a + b; }
inline double gqc_sub(double a, double b) { return a - b; }
inline double gqc_mul(double a, double b) { return a * b; }
inline double gqc_div(double a, double b) { return a / b; }
inline double gqc_fma(double a, double b, double c) { return std::fma(a, b, c); }
inline double gqc_rcp(double a) { return 1.0 / a; }
inline double gqc_floor(double a) { return std::floor(a); }
inline long long gqc_bits(double a) {
    long long b;
    std::memcpy(&b, &a, sizeof b);
    return b;
}
inline int gqc_ffsll(long long a) { return __builtin_ffsll(a); }
inline int gqc_max(int a, int b) { return a > b ? a : b; }
inline bool gqc_lo_odd(double a) { return gqc_bits(a) & 1; }
inline int exp_field(double x) { return static_cast<int>((gqc_bits(x) >> 52) & 0x7ff); }
inline double pow2_field(int f) {
    const long long b = static_cast<long long>(f) << 52;
    double d;
    std::memcpy(&d, &b, sizeof d);
    return d;
}
#endif

// ---------------------------------------------------------------------------
// Exact fast-forward of L sequential adds s <- fl(s + c), s >= 0, c >= 0.
//
// Inside a binade [base, 2 base) of s (unit in the last place u = base*2^-52;
// the subnormals share u = 2^-1074 with [2^-1022, 2^-1021) and are treated as
// that binade), an add whose exact result stays <= 2 base rounds on the
// u-grid, so fl(s + c) = s + inc with inc = round_u(c). round_u(c) can depend
// on the parity of s/u only when c is an exact half-ulp tie (for a given c
// that happens in exactly one binade, f_tie), and a tie always lands on an
// even multiple, after which the increment is constant. inc is read off an
// even reference point, inc = fl(base + c) - base; an odd s in the tie binade
// takes one real step first. A run that ends inside the binade is one exact
// fma (s + L*inc lies on the u-grid below 2 base). A run that reaches the top
// jumps the m = floor((2 base - u - s) / inc) steps that provably stay inside
// (their exact sums stay below 2 base - u/2), then crosses with one real add.
// c >= base/2 (at most two adds per binade) is stepped with real adds, and
// inc == 0 (c <= u/2) is a fixed point after at most one real add.
//
// A Chain caches the binade parameters of its partial sum, so runs that stay
// inside a binade (the common case once the sum is large) cost one fma and
// the per-binade work is paid once per crossing. The state is kept minimal
// (three doubles and two ints) because the kernel holds two chains per thread
// and its occupancy is register-bound.
// ---------------------------------------------------------------------------
struct Chain {
    double s;    // partial sum
    double top;  // 2 base of the cached binade (0: no cache)
    double inc;  // settled increment in the cached binade
    int f_tie;   // binade in which c is a half-ulp tie
    int flags;   // bit 0: c < base/2 (jumpable); bit 1: cached binade == f_tie
};
constexpr int kJump = 1;
constexpr int kTie = 2;

// Biased exponent f of the binade whose half-ulp is the lowest set bit of c.
GQC_HD inline int tie_binade(const double c) {
    const long long bits = gqc_bits(c);
    int e = static_cast<int>((bits >> 52) & 0x7ff);
    long long mant = bits & ((1ll << 52) - 1);
    if (e > 0) mant |= (1ll << 52);
    else e = 1;
    return e + gqc_ffsll(mant);  // e + 1 + (index of the lowest set bit)
}

GQC_HD inline Chain make_chain(const double s, const double c) {
    Chain ch;
    ch.s = s;
    ch.top = 0.0;
    ch.inc = 0.0;
    ch.f_tie = tie_binade(c);
    ch.flags = 0;
    return ch;
}

GQC_HD inline void refresh(Chain& ch, const double c) {
    const int f = gqc_max(exp_field(ch.s), 1);
    const double base = pow2_field(f);
    ch.top = gqc_add(base, base);
    const bool jump = c < gqc_mul(base, 0.5);
    ch.inc = jump ? gqc_sub(gqc_add(base, c), base) : 0.0;
    ch.flags = (jump ? kJump : 0) | (f == ch.f_tie ? kTie : 0);
}

// In-binade fast path is allowed: jumpable and not (tie binade with odd s).
GQC_HD inline bool settled(const Chain& ch) {
    return (ch.flags & kJump) && !((ch.flags & kTie) && gqc_lo_odd(ch.s));
}

// Exact jump count of the slow path: the largest m with s + m*inc <= top - u.
// The true quotient is < L <= 2^31 wherever this is called, so the estimate is
// off by at most one and the two fma sign tests (exact: room - m*inc is a
// u-grid multiple) settle it. Tiny binades (1/inc would overflow) divide.
GQC_HD inline double max_steps(const Chain& ch, const double room) {
    const double q = ch.top > 0x1p-950 ? gqc_mul(room, gqc_rcp(ch.inc)) : gqc_div(room, ch.inc);
    double m = gqc_floor(q);
    if (gqc_fma(-m, ch.inc, room) < 0.0) m = m - 1.0;
    else if (gqc_fma(-(m + 1.0), ch.inc, room) >= 0.0) m = m + 1.0;
    return m;
}

GQC_HD inline double room_of(const Chain& ch) {
    const double u = gqc_mul(ch.top, 0x1p-53);
    return gqc_sub(gqc_sub(ch.top, u), ch.s);
}

// L sequential adds of c (the general loop).
GQC_HD inline void ff_run(Chain& ch, const double c, int L) {
    while (L > 0) {
        if (!(ch.s < ch.top)) refresh(ch, c);
        if (!(ch.flags & kJump)) {  // c >= base/2: real adds
            ch.s = gqc_add(ch.s, c);
            --L;
            continue;
        }
        if (ch.inc == 0.0) {  // c <= u/2: fixed point after one add
            ch.s = gqc_add(ch.s, c);
            return;
        }
        if ((ch.flags & kTie) && gqc_lo_odd(ch.s)) {  // settle tie parity
            ch.s = gqc_add(ch.s, c);
            --L;
            continue;
        }
        const double t = gqc_fma(static_cast<double>(L), ch.inc, ch.s);
        if (t < ch.top) {  // the whole remainder stays in the binade: exact
            ch.s = t;
            return;
        }
        const double m = max_steps(ch, room_of(ch));
        ch.s = gqc_fma(m, ch.inc, ch.s);  // exact: a u-grid point below 2 base
        L -= static_cast<int>(m);
        ch.s = gqc_add(ch.s, c);  // crosses into the next binade
        --L;
    }
}

// One pass over a run of L > 0 adds that handles up to one binade crossing
// inline: the whole run if it stays in the binade (one exact fma; inc == 0 is
// the fixed point t == s), else the maximal in-binade jump plus the crossing
// add (or a single real add when c >= base/2 or at a half-ulp tie with odd
// s), then the remainder in the new binade if it fits there. Leaves L > 0
// only for runs that cross more than one binade.
GQC_HD inline void ff_pass(Chain& ch, const double c, int& L) {
    if (!(ch.s < ch.top)) refresh(ch, c);
    const bool ok = settled(ch);
    const double t = gqc_fma(static_cast<double>(L), ch.inc, ch.s);
    if (ok && t < ch.top) {
        ch.s = t;
        L = 0;
        return;
    }
    const double m = ok ? max_steps(ch, room_of(ch)) : 0.0;
    const double top = ch.top;
    ch.s = gqc_add(gqc_fma(m, ch.inc, ch.s), c);
    L -= static_cast<int>(m) + 1;
    if (ok) {
        // a settled crossing lands in the next binade [top, 2 top): the exact
        // sum is below top + c and c < base/2 = top/4; c stays jumpable there
        ch.top = gqc_add(top, top);
        ch.inc = gqc_sub(gqc_add(top, c), top);
        ch.flags = kJump | (exp_field(top) == ch.f_tie ? kTie : 0);
    } else {
        refresh(ch, c);  // a single real add (c >= base/2, or an odd tie)
    }
    if (L <= 0) return;
    const double t2 = gqc_fma(static_cast<double>(L), ch.inc, ch.s);
    if (settled(ch) && t2 < ch.top) {
        ch.s = t2;
        L = 0;
    }
}

// Both chains of a W run of length L > 0: one pass each (independent, so the
// two dependency chains interleave), then the general loop for the rare runs
// that cross several binades.
GQC_HD inline void ff_run2(Chain& a, const double ca, Chain& b, const double cb, const int L) {
    int La = L, Lb = L;
    ff_pass(a, ca, La);
    ff_pass(b, cb, Lb);
    if (La > 0) ff_run(a, ca, La);
    if (Lb > 0) ff_run(b, cb, Lb);
}

// One step of a W run for ff_walk2: either the whole remainder inside the
// binade (returns with L = 0), or the maximal in-binade jump plus the crossing
// add and an incremental refresh (settled chains), or one real add (c >=
// base/2, or the odd side of a half-ulp tie). Every branch consumes >= 1 add.
GQC_HD inline void ff_step(Chain& ch, const double c, int& L) {
    // the fma is issued before the flag/parity test so its latency overlaps
    // it (measured: 4.75 -> 4.54 ms on LFR 1M x 32)
    const double t = gqc_fma(static_cast<double>(L), ch.inc, ch.s);
    const bool ok = settled(ch);
    if (ok && t < ch.top) {
        ch.s = t;
        L = 0;
        return;
    }
    if (ok) {
        const double m = max_steps(ch, room_of(ch));
        const double top = ch.top;
        ch.s = gqc_add(gqc_fma(m, ch.inc, ch.s), c);
        L -= static_cast<int>(m) + 1;
        ch.top = gqc_add(top, top);  // landed in [top, 2 top): see ff_pass
        ch.inc = gqc_sub(gqc_add(top, c), top);
        ch.flags = kJump | (exp_field(top) == ch.f_tie ? kTie : 0);
#if GQC_STEP_FINISH
        // finish the run in the new binade when it fits (a single-crossing
        // run then costs one trip of ff_walk2's loop instead of two)
        if (L > 0 && settled(ch)) {
            const double t2 = gqc_fma(static_cast<double>(L), ch.inc, ch.s);
            if (t2 < ch.top) {
                ch.s = t2;
                L = 0;
            }
        }
#endif
    } else {
        ch.s = gqc_add(ch.s, c);
        --L;
        refresh(ch, c);
    }
}

// Both chains of a W run of length L > 0 in one loop: the warp iterates
// 1 + (most binade crossings of any lane and chain) times over one compact
// body instead of a pass per chain plus the general loop for multi-crossings.
// Cache refresh at the start of a W run. A neighbour add that crossed the
// cached binade of a jumpable chain lands in the next one (the add is below
// base/2 < top), so the cache moves up one binade incrementally, as after a
// settled crossing in ff_step; anything else recomputes it.
GQC_HD inline void refresh_after_add(Chain& ch, const double c) {
#if GQC_INCR_REFRESH
    if ((ch.flags & kJump) && ch.s < gqc_add(ch.top, ch.top)) {
        const double base = ch.top;
        ch.top = gqc_add(base, base);
        ch.inc = gqc_sub(gqc_add(base, c), base);
        ch.flags = kJump | (exp_field(base) == ch.f_tie ? kTie : 0);
        return;
    }
#endif
    refresh(ch, c);
}

GQC_HD inline void ff_walk2(Chain& a, const double ca, Chain& b, const double cb, const int L) {
    if (!(a.s < a.top)) refresh_after_add(a, ca);
    if (!(b.s < b.top)) refresh_after_add(b, cb);
    int La = L, Lb = L;
    do {
        if (La > 0) ff_step(a, ca, La);
        if (Lb > 0) ff_step(b, cb, Lb);
    } while (La > 0 || Lb > 0);
}

// ---------------------------------------------------------------------------
// Batched walk over neighbour events (unit weights). Event q of a chunk is the
// run of W terms over columns [pos, col(q)) followed by one neighbour term c1
// at column col(q) (columns strictly ascending, pos <= col(first)). Inside a
// binade [base, top) of s in which both c and c1 are jumpable (< base/2) and
// neither is a half-ulp tie, every add is an exact u-grid increment, so the
// sum after event q is exactly
//     s + A(q) * inc + B(q) * inc1,   A = W columns up to col(q), B = events,
// as long as that value stays below top (two exact fmas; the "< top" test is
// exact even when it fails because rounding is monotone). The value is
// monotone in q, so a binary search finds the last event that stays in the
// binade; everything before it is applied at once and the next event crosses
// (with max_steps inside its W run, or at its neighbour add). Binades where
// the batch rule does not hold are walked one event at a time with ff_run.
// The work per chunk is O((crossings + 1) * log(events)) instead of one
// fast-forward per event.
// ---------------------------------------------------------------------------
#ifndef GQC_WALK_COUNT
#define GQC_WALK_COUNT()
#endif
// One accumulator's position in a batched walk: sum s, next event e, first
// column not yet added pos.
struct WalkState {
    double s;
    int e, pos;
};

// One iteration of the batched walk: everything up to the next binade
// crossing (or the range's end) plus that crossing event.
template <class Cols>
GQC_HD inline void walk_step(WalkState& w, const double c, const double c1, const int tie_c, const int tie_c1,
                             const Cols& col, const int end) {
    GQC_WALK_COUNT();
    double s = w.s;
    int e = w.e, pos = w.pos;
    const int f = gqc_max(exp_field(s), 1);
    const double base = pow2_field(f);
    const double top = gqc_add(base, base);
    const double half = gqc_mul(base, 0.5);
    if (c < half && c1 < half && f != tie_c && f != tie_c1) {
        const double inc = gqc_sub(gqc_add(base, c), base);
        const double inc1 = gqc_sub(gqc_add(base, c1), base);
        int lo = e - 1, hi = end - 1;  // last event whose sum stays below top (e - 1: none)
        {  // common case: the rest of the range stays in the binade
            const double t = gqc_fma(static_cast<double>(end - e), inc1,
                                     gqc_fma(static_cast<double>(col(end - 1) - pos - (end - 1 - e)), inc, s));
            if (t < top) lo = hi;
        }
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            const double t = gqc_fma(static_cast<double>(mid - e + 1), inc1,
                                     gqc_fma(static_cast<double>(col(mid) - pos - (mid - e)), inc, s));
            if (t < top) lo = mid;
            else hi = mid - 1;
        }
        if (lo >= e) {
            const int cl = col(lo);
            s = gqc_fma(static_cast<double>(lo - e + 1), inc1,
                        gqc_fma(static_cast<double>(cl - pos - (lo - e)), inc, s));
            pos = cl + 1;
            e = lo + 1;
            if (e == end) {
                w.s = s;
                w.e = e;
                w.pos = pos;
                return;
            }
        }
        // event e leaves the binade: inside its W run or at its neighbour add
        const int ce = col(e);
        const int L = ce - pos;
        const double t = gqc_fma(static_cast<double>(L), inc, s);
        if (t < top) {
            s = t;
        } else {
            Chain ch;
            ch.s = s;
            ch.top = top;
            ch.inc = inc;
            ch.f_tie = tie_c;
            ch.flags = kJump;
            const double m = max_steps(ch, room_of(ch));
            ch.s = gqc_add(gqc_fma(m, inc, s), c);
            ch.top = 0.0;
            ff_run(ch, c, L - static_cast<int>(m) - 1);
            s = ch.s;
        }
        s = gqc_add(s, c1);
        pos = ce + 1;
        ++e;
    } else {  // one event at a time (tiny sums, tie binades)
        const int ce = col(e);
        if (ce > pos) {
            Chain ch = make_chain(s, c);
            ch.f_tie = tie_c;
            ff_run(ch, c, ce - pos);
            s = ch.s;
        }
        s = gqc_add(s, c1);
        pos = ce + 1;
        ++e;
    }
    w.s = s;
    w.e = e;
    w.pos = pos;
}

template <class Cols>
GQC_HD inline double walk_events(double s, const double c, const double c1, const int tie_c, const int tie_c1,
                                 const Cols& col, int e, const int end, int pos) {
    WalkState w{s, e, pos};
    while (w.e < end) walk_step(w, c, c1, tie_c, tie_c1, col, end);
    return w.s;
}

// Both accumulators of a row over events [e, end) in one loop: the warp
// iterates max(crossings) times over the two chains instead of the sum of
// two walks, and the two dependency chains interleave.
template <class Cols>
GQC_HD inline void walk_events2(double& sa, const double ca, const double c1a, const int ta, const int t1a, double& sb,
                                const double cb, const double c1b, const int tb, const int t1b, const Cols& col,
                                const int e, const int end, const int pos) {
    WalkState a{sa, e, pos}, b{sb, e, pos};
    while (a.e < end || b.e < end) {
        if (a.e < end) walk_step(a, ca, c1a, ta, t1a, col, end);
        if (b.e < end) walk_step(b, cb, c1b, tb, t1b, col, end);
    }
    sa = a.s;
    sb = b.s;
}

// ---------------------------------------------------------------------------
// Batched walk over events of NC classes (the k-hop extension: class h = a
// hop-h term). Same rule as walk_events with one increment per class: inside
// a binade where c and every class constant cc[k] are jumpable and none is a
// half-ulp tie there, the sum after event q is exactly
//     s + A(q) * inc + sum_k B_k(q) * inc_k,
// A = W columns in [pos, col(q)), B_k = class-k events in [e, q]. Every
// partial value of the fma chain is a u-grid point no larger than the final
// one, so all are exact while the final stays below top, and monotone
// rounding keeps the "< top" test exact when it does not. Ev provides
// col(q), cls(q) in [0, NC) and cnt(q, k) = class-k events among [0, q] of
// the current chunk (cnt(-1, k) = 0).
// ---------------------------------------------------------------------------
template <int NC, class Ev>
GQC_HD inline double walk_events_multi(double s, const double c, const int tie_c, const double* cc,
                                       const int* tie_cc, const Ev& ev, int e, const int end, int pos) {
    while (e < end) {
        GQC_WALK_COUNT();
        const int f = gqc_max(exp_field(s), 1);
        const double base = pow2_field(f);
        const double top = gqc_add(base, base);
        const double half = gqc_mul(base, 0.5);
        bool ok = c < half && f != tie_c;
#pragma unroll
        for (int k = 0; k < NC; ++k) ok = ok && cc[k] < half && f != tie_cc[k];
        if (ok) {
            const double inc = gqc_sub(gqc_add(base, c), base);
            double inck[NC];
            int b0[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                inck[k] = gqc_sub(gqc_add(base, cc[k]), base);
                b0[k] = ev.cnt(e - 1, k);
            }
            auto value = [&](const int q) {
                double t = gqc_fma(static_cast<double>(ev.col(q) - pos - (q - e)), inc, s);
#pragma unroll
                for (int k = 0; k < NC; ++k) t = gqc_fma(static_cast<double>(ev.cnt(q, k) - b0[k]), inck[k], t);
                return t;
            };
            int lo = e - 1, hi = end - 1;  // last event whose sum stays below top (e - 1: none)
            if (value(hi) < top) lo = hi;  // common case: the rest of the range stays in the binade
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (value(mid) < top) lo = mid;
                else hi = mid - 1;
            }
            if (lo >= e) {
                s = value(lo);
                pos = ev.col(lo) + 1;
                e = lo + 1;
                if (e == end) break;
            }
            // event e leaves the binade: inside its W run or at its own term
            const int ce = ev.col(e);
            const int L = ce - pos;
            const double t = gqc_fma(static_cast<double>(L), inc, s);
            if (t < top) {
                s = t;
            } else {
                Chain ch;
                ch.s = s;
                ch.top = top;
                ch.inc = inc;
                ch.f_tie = tie_c;
                ch.flags = kJump;
                const double m = max_steps(ch, room_of(ch));
                ch.s = gqc_add(gqc_fma(m, inc, s), c);
                ch.top = 0.0;
                ff_run(ch, c, L - static_cast<int>(m) - 1);
                s = ch.s;
            }
            s = gqc_add(s, cc[ev.cls(e)]);
            pos = ce + 1;
            ++e;
        } else {  // one event at a time (tiny sums, tie binades)
            const int ce = ev.col(e);
            if (ce > pos) {
                Chain ch = make_chain(s, c);
                ch.f_tie = tie_c;
                ff_run(ch, c, ce - pos);
                s = ch.s;
            }
            s = gqc_add(s, cc[ev.cls(e)]);
            pos = ce + 1;
            ++e;
        }
    }
    return s;
}

// ---------------------------------------------------------------------------
// Prefix segments of the pure trajectory P(t) = t sequential adds of c from
// s = 0 (every row's first run, before its first neighbour or itself, is such
// a run). Segment k covers [t[k], t[k+1]) with P(t) = s0[k] + (t - t[k])*inc[k]
// exactly (inc 0 for single real steps and for the final fixed point). The
// builder follows ff_run step for step; from t_end on the caller continues
// from s_end with ff_run.
// ---------------------------------------------------------------------------
constexpr int kPrefixCap = 96;
constexpr int kPrefixForever = 0x7fffffff;

GQC_HD inline void build_prefix(const double c, const int n, int* t_out, double* s_out, double* inc_out,
                                int* count, int* t_end, double* s_end) {
    Chain ch = make_chain(0.0, c);
    int t = 0, k = 0;
    while (t < n && k < kPrefixCap - 1) {
        if (!(ch.s < ch.top)) refresh(ch, c);
        if (!(ch.flags & kJump) || (ch.inc != 0.0 && !settled(ch))) {  // single real step
            t_out[k] = t;
            s_out[k] = ch.s;
            inc_out[k] = 0.0;
            ++k;
            ch.s = gqc_add(ch.s, c);
            ++t;
            continue;
        }
        if (ch.inc == 0.0) {  // one add, then a fixed point forever
            t_out[k] = t;
            s_out[k] = ch.s;
            inc_out[k] = 0.0;
            ++k;
            ch.s = gqc_add(ch.s, c);
            ++t;
            t_out[k] = t;
            s_out[k] = ch.s;
            inc_out[k] = 0.0;
            ++k;
            t = kPrefixForever;
            break;
        }
        double m = max_steps(ch, room_of(ch));
        if (m > static_cast<double>(n - t)) m = static_cast<double>(n - t);
        t_out[k] = t;  // valid for [t, t + m]
        s_out[k] = ch.s;
        inc_out[k] = ch.inc;
        ++k;
        ch.s = gqc_fma(m, ch.inc, ch.s);
        t += static_cast<int>(m);
        if (t >= n) break;
        ch.s = gqc_add(ch.s, c);  // crossing
        ++t;
    }
    *count = k;
    *t_end = t;
    *s_end = ch.s;
}

// P(L) for 0 <= L < t_end, by binary search for the last segment start <= L.
GQC_HD inline double prefix_value(const int* t, const double* s0, const double* inc, const int count, const int L) {
    int lo = 0, hi = count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (t[mid] <= L) lo = mid;
        else hi = mid - 1;
    }
    return gqc_fma(static_cast<double>(L - t[lo]), inc[lo], s0[lo]);
}

}  // namespace ffc
}  // namespace gqc

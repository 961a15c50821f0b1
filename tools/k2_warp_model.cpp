// Warp-level model of potential_warp_kernel's per-event path (non-batched rows):
// 32 sigma lanes x 2 chains walk the row's events through ff_walk2/ff_step;
// counts, per event, whether ANY lane enters each branch (the warp executes it).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>
#include "../paper_2305_14641_b200/csrc/ff_chain.cuh"
using namespace gqc::ffc;

struct Counters { long long events = 0, trips = 0, entry_refresh = 0, step_fast = 0, step_cross = 0, step_real = 0, lane_cross = 0, lane_real = 0, lane_refresh = 0; };

extern "C" void sim_rows(const long long* off, const int* nbr, const int* rows, int nrows, int n,
                         const double* pW, const double* eW, const double* p1, const double* e1, int S,
                         long long* out) {
    Counters C;
    for (int r = 0; r < nrows; ++r) {
        const int i = rows[r];
        const long long kb = off[i], ke = off[i + 1];
        if (ke - kb >= 32) continue;  // batched rows are not modelled
        std::vector<Chain> num(S), den(S);
        for (int s = 0; s < S; ++s) { num[s] = make_chain(0.0, pW[s]); den[s] = make_chain(0.0, eW[s]); }
        // events: neighbours and self, in column order; runs between them
        std::vector<int> ev;
        bool self_done = false;
        for (long long k = kb; k <= ke; ++k) {
            const int col = k < ke ? nbr[k] : n;
            if (!self_done && i < col) { ev.push_back(-1 - i); self_done = true; }
            if (k < ke) ev.push_back(col);
        }
        int pos = 0;
        bool first = true;
        for (size_t q = 0; q <= ev.size(); ++q) {
            const bool self = q < ev.size() && ev[q] < 0;
            const int col = q < ev.size() ? (self ? -1 - ev[q] : ev[q]) : n;
            const int L = col - pos;
            if (L > 0) {
                if (first) {  // prefix table (not modelled): exact pure trajectory
                    for (int s = 0; s < S; ++s) {
                        ff_run(num[s], pW[s], L); num[s].top = 0.0;
                        ff_run(den[s], eW[s], L); den[s].top = 0.0;
                    }
                } else {
                    ++C.events;
                    // ff_walk2: entry refresh, then trips
                    bool any_ref = false;
                    for (int s = 0; s < S; ++s) {
                        if (!(num[s].s < num[s].top)) { refresh(num[s], pW[s]); any_ref = true; ++C.lane_refresh; }
                        if (!(den[s].s < den[s].top)) { refresh(den[s], eW[s]); any_ref = true; ++C.lane_refresh; }
                    }
                    C.entry_refresh += any_ref;
                    std::vector<int> La(S, L), Lb(S, L);
                    for (;;) {
                        bool any = false, f = false, cr = false, re = false;
                        for (int s = 0; s < S; ++s) {
                            for (int c2 = 0; c2 < 2; ++c2) {
                                Chain& ch = c2 ? den[s] : num[s];
                                int& Lx = c2 ? Lb[s] : La[s];
                                const double cc = c2 ? eW[s] : pW[s];
                                if (Lx <= 0) continue;
                                any = true;
                                const double t = std::fma((double)Lx, ch.inc, ch.s);
                                const bool ok = settled(ch);
                                if (ok && t < ch.top) { f = true; ch.s = t; Lx = 0; continue; }
                                if (ok) { cr = true; ++C.lane_cross; ff_step(ch, cc, Lx); }
                                else { re = true; ++C.lane_real; ff_step(ch, cc, Lx); }
                            }
                        }
                        if (!any) break;
                        ++C.trips; C.step_fast += f; C.step_cross += cr; C.step_real += re;
                    }
                }
            }
            first = false;
            if (q == ev.size()) break;
            for (int s = 0; s < S; ++s) {
                if (self) den[s].s = den[s].s + 1.0;
                else { num[s].s = num[s].s + p1[s]; den[s].s = den[s].s + e1[s]; }
            }
            pos = col + 1;
        }
    }
    long long* o = out;
    o[0] = C.events; o[1] = C.trips; o[2] = C.entry_refresh; o[3] = C.step_fast; o[4] = C.step_cross; o[5] = C.step_real;
    o[6] = C.lane_cross; o[7] = C.lane_real; o[8] = C.lane_refresh;
}

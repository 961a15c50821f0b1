// Host-side unit tests of the graphqc-compatible facade (CPU, no device):
// the reference's graph/metrics/sweep test cases (tests/graph_test.cpp,
// metrics_test.cpp, sweep_test.cpp in the reference) that do not need a
// potential field. Built and run by tests/test_facade.py.
#include <cmath>
#include <cstdint>
#include <iostream>
#include <map>
#include <random>
#include <vector>
#include <sstream>
#include <string>
#include <tuple>

#include "graphqc/format.hpp"
#include "graphqc/ggd.hpp"
#include "graphqc/graph.hpp"
#include "graphqc/metrics.hpp"
#include "graphqc/sweep.hpp"

using namespace graphqc;

static int failures = 0;
#define CHECK(cond)                                                                 \
    do {                                                                            \
        if (!(cond)) {                                                              \
            ++failures;                                                             \
            std::cerr << __FILE__ << ":" << __LINE__ << ": CHECK failed: " #cond "\n"; \
        }                                                                           \
    } while (0)
#define CHECK_THROWS(expr, type)                    \
    do {                                            \
        bool thrown = false;                        \
        try {                                       \
            (void)(expr);                           \
        } catch (const type&) {                     \
            thrown = true;                          \
        } catch (...) {                             \
        }                                           \
        if (!thrown) {                              \
            ++failures;                             \
            std::cerr << __FILE__ << ":" << __LINE__ \
                      << ": expected " #type "\n";  \
        }                                           \
    } while (0)

static Graph from_text(const std::string& text, double w = 10.0) {
    std::istringstream in(text);
    return parse_edge_list(in, w, "<test>");
}

static std::string what_of(const std::string& text) {
    try {
        from_text(text);
    } catch (const std::exception& e) {
        return e.what();
    }
    return "";
}

// graph.cpp:25-71 restated the slow way (a std::map per row, keep-first
// collapse in input order): the CSR the facade's multi-threaded host build
// must reproduce byte for byte.
static bool csr_matches_map_build(std::int32_t n, const std::vector<Edge>& edges) {
    std::vector<std::map<std::int32_t, double>> rows(n);
    for (const Edge& e : edges) {
        if (e.u == e.v) continue;
        if (rows[e.u].count(e.v)) continue;  // keep-first
        rows[e.u][e.v] = e.weight;
        rows[e.v][e.u] = e.weight;
    }
    Graph g(n, std::span<const Edge>(edges), 10.0);
    const Graph::CsrView c = g.csr();
    std::int64_t k = 0;
    bool unit = true;
    for (std::int32_t i = 0; i < n; ++i) {
        if (c.offsets[i] != k) return false;
        for (const auto& [j, w] : rows[i]) {
            if (c.nbr[k] != j || c.weights[k] != w) return false;
            unit = unit && w == 1.0;
            ++k;
        }
    }
    return c.offsets[n] == k && c.unit == unit;
}

int main(int argc, char** argv) {
    const std::string data = argc > 1 ? argv[1] : "tests/golden";
    // the host CSR build with many threads (>= 2^18 edges): random weighted
    // edges with duplicates in both orientations (some with another weight)
    // and self loops, and a unit-weight variant
    {
        std::mt19937_64 rng(7);
        const std::int32_t n = 50000;
        const std::size_t m = 400000;
        std::vector<Edge> e(m);
        const double ws[4] = {0.5, 1.0, 1.5, 2.0};
        for (auto& x : e) x = {static_cast<std::int32_t>(rng() % n), static_cast<std::int32_t>(rng() % n), ws[rng() % 4]};
        for (std::size_t q = 0; q < m / 20; ++q) {  // re-emit earlier pairs
            const Edge& s = e[rng() % m];
            Edge& d = e[rng() % m];
            d = (rng() & 1) ? Edge{s.v, s.u, ws[rng() % 4]} : Edge{s.u, s.v, s.weight};
        }
        for (std::size_t q = 0; q < m / 100; ++q) {  // self loops
            Edge& x = e[rng() % m];
            x.v = x.u;
        }
        CHECK(csr_matches_map_build(n, e));
        for (auto& x : e) x.weight = 1.0;
        CHECK(csr_matches_map_build(n, e));
    }
    // graph_test.cpp: parsing builds a symmetric unit-weight graph
    {
        Graph g = from_text("a b\nb c\n");
        CHECK(g.num_nodes() == 3 && g.num_edges() == 2 && g.default_distance() == 10.0);
        CHECK(g.name_of(0) == "a" && g.id_of("c") == 2 && g.id_of("zz") == -1);
        auto nb = neighbors(g, 1);
        CHECK(nb.size() == 2 && nb[0] == std::make_pair(0, 1.0) && nb[1] == std::make_pair(2, 1.0));
        CHECK(g.csr().unit);
    }
    // duplicates collapse; a conflicting duplicate keeps the first weight
    {
        Graph g = from_text("1 2 2.5\n2 1 2.5\n");
        CHECK(g.num_nodes() == 2 && g.num_edges() == 1 && pairwise_distance(g, 0, 1) == 2.5);
        Graph h = from_text("a b 1.5\nb a 2.5\n");
        CHECK(h.num_edges() == 1 && pairwise_distance(h, 0, 1) == 1.5 && !h.csr().unit);
    }
    // self loops dropped (names still interned)
    {
        Graph g = from_text("a a\na b\n");
        CHECK(g.num_nodes() == 2 && g.num_edges() == 1 && neighbors(g, 0).size() == 1);
    }
    // modularity(g, assignment) always recomputes from the graph it is given
    // (metrics.cpp:37-44): the device intra count is private to run_sweep
    {
        Graph g = from_text("0 1\n1 2\n2 0\n3 4\n4 5\n5 3\n2 3\n");
        ClusterAssignment a;
        a.cluster_index = {0, 0, 0, 1, 1, 1};
        a.num_clusters = 2;
        CHECK(modularity(g, a) == modularity(g, std::span<const std::int32_t>(a.cluster_index)));
        Graph h = from_text("0 1\n1 2\n2 0\n3 4\n4 5\n5 3\n0 3\n1 4\n");
        CHECK(modularity(h, a) != modularity(g, a));
    }
    // parse errors carry the line number
    CHECK(what_of("a b\nx\n").find("line 2") != std::string::npos);
    CHECK(what_of("a b 0\n").find("non-positive") != std::string::npos);
    CHECK(what_of("a b -1\n").find("non-positive") != std::string::npos);
    CHECK(what_of("a b x\n").find("weight") != std::string::npos);
    CHECK_THROWS(from_text("# only comments\n\n"), IoError);
    CHECK_THROWS(from_text("a b\n", 0.0), std::invalid_argument);
    // pairwise distance
    {
        Graph g = from_text("a b 2.0\nb c\n", 10.0);
        CHECK(pairwise_distance(g, 0, 1) == 2.0 && pairwise_distance(g, 0, 2) == 10.0 && pairwise_distance(g, 1, 1) == 0.0);
        CHECK_THROWS(pairwise_distance(g, 0, 7), std::out_of_range);
    }
    // isolated node; graph ctor validation
    {
        Graph g(3, std::vector<Edge>{{0, 1, 1.0}}, 10.0);
        CHECK(neighbors(g, 2).empty() && g.degree(2) == 0);
        CHECK_THROWS(Graph(0, std::vector<Edge>{}, 10.0), std::invalid_argument);
        CHECK_THROWS(Graph(2, std::vector<Edge>{{0, 5, 1.0}}, 10.0), std::out_of_range);
        CHECK_THROWS(Graph(2, std::vector<Edge>{{0, 1, 0.0}}, 10.0), std::invalid_argument);
        CHECK_THROWS(g.degree(3), std::out_of_range);
    }
    // round trip through the text form
    {
        std::vector<Edge> edges;
        for (int i = 0; i + 1 < 40; ++i) edges.push_back({i, i + 1, 1.0});
        edges.push_back({3, 17, 0.75});
        edges.push_back({17, 3, 0.5});  // conflicting duplicate: first kept (and warned)
        Graph g(40, edges, 10.0);
        std::ostringstream out;
        write_edge_list(out, g);
        Graph h = from_text(out.str(), g.default_distance());
        CHECK(h.num_nodes() == g.num_nodes() && h.num_edges() == g.num_edges());
        CHECK(pairwise_distance(h, h.id_of("3"), h.id_of("17")) == 0.75);
    }
    // labels
    {
        Graph g = from_text("a b\nb c\n");
        std::istringstream two("a x\nb y\nc x\n");
        LabelSet ls = parse_labels(two, g, "<test>");
        CHECK(ls.num_classes() == 2 && ls.label_of(0) == 0 && ls.label_of(1) == 1 && ls.label_of(2) == 0);
        std::istringstream missing("a x\nb y\n");
        CHECK_THROWS(parse_labels(missing, g, "<test>"), IoError);
        std::istringstream unknown("a x\nb y\nc x\nq x\n");
        CHECK_THROWS(parse_labels(unknown, g, "<test>"), IoError);
        std::istringstream conflict("a x\na y\nb x\nc x\n");
        CHECK_THROWS(parse_labels(conflict, g, "<test>"), IoError);
        std::istringstream repeat("a x\na x\nb y\nc x\n");
        CHECK(parse_labels(repeat, g, "<test>").num_classes() == 2);
    }
    // integer names (value -> id array instead of a hash map): ids follow first
    // appearance, and only the canonical spelling of a name is that name
    {
        Graph g = from_text("7 3\n3 100\n0 7\n");
        CHECK(g.num_nodes() == 4 && g.id_of("7") == 0 && g.id_of("3") == 1 && g.id_of("100") == 2 && g.id_of("0") == 3);
        CHECK(g.id_of("07") == -1 && g.id_of("+7") == -1 && g.id_of("5") == -1 && g.id_of("101") == -1 &&
              g.id_of("99999999999") == -1 && g.id_of("") == -1 && g.id_of("a") == -1);
        std::istringstream ok("0 p\n3 q\n7 p\n100 q\n");
        CHECK(parse_labels(ok, g, "<test>").label_of(g.id_of("100")) == 1);
        std::istringstream padded("0 p\n3 q\n07 p\n100 q\n");
        CHECK_THROWS(parse_labels(padded, g, "<test>"), IoError);
        Graph mixed = from_text("7 3\n07 x\n");  // "07" is its own node next to "7"
        CHECK(mixed.num_nodes() == 4 && mixed.id_of("07") == 2 && mixed.id_of("7") == 0);
    }
    // karate fixture shape (graph_test.cpp:165-178)
    {
        Graph g = load_edge_list(data + "/karate.edges", 10.0);
        CHECK(g.num_nodes() == 34 && g.num_edges() == 78);
        CHECK(neighbors(g, g.id_of("0")).size() == 16 && neighbors(g, g.id_of("33")).size() == 17);
        LabelSet ls = load_labels(data + "/karate.labels", g);
        int sizes[2] = {0, 0};
        for (int i = 0; i < g.num_nodes(); ++i) ++sizes[ls.label_of(i)];
        CHECK(ls.num_classes() == 2 && sizes[0] == 17 && sizes[1] == 17);
        // karate ground-truth modularity (acceptance criterion 3 value)
        std::vector<std::int32_t> split(ls.labels().begin(), ls.labels().end());
        CHECK(std::abs(modularity(g, split)) < 1.0 && modularity(g, split) > 0.3);
        CHECK_THROWS(load_edge_list(data + "/no_such.edges", 10.0), IoError);
    }
    // components, complete graph
    {
        Graph g = from_text("a b\nb c\nx y\n");
        auto [comp, count] = connected_components(g);
        CHECK(count == 2 && comp[g.id_of("a")] == comp[g.id_of("c")] && comp[g.id_of("x")] != comp[g.id_of("a")]);
        std::vector<Edge> edges;
        for (int i = 0; i < 5; ++i)
            for (int j = i + 1; j < 5; ++j) edges.push_back({i, j, 1.0});
        Graph a(5, edges, 10.0), b = complete_graph(5);
        CHECK(a.num_edges() == b.num_edges());
        for (int i = 0; i < 5; ++i) CHECK(neighbors(a, i) == neighbors(b, i));
    }
    // metrics_test.cpp basics
    {
        auto t = contingency(std::vector<int>{0, 0, 1, 1}, 2, std::vector<int>{0, 0, 0, 1}, 2);
        CHECK(t.count(0, 0) == 2 && t.count(0, 1) == 0 && t.count(1, 0) == 1 && t.count(1, 1) == 1);
        CHECK(t.row_sums[0] == 2 && t.col_sums[0] == 3 && t.total == 4);
        CHECK(ari(contingency(std::vector<int>{0, 0, 1, 1}, 2, std::vector<int>{1, 1, 0, 0}, 2)) == 1.0);
        CHECK(ari(t) == 0.0);
        CHECK_THROWS(ari(contingency(std::vector<int>{0}, 1, std::vector<int>{0}, 1)), std::invalid_argument);
        CHECK(ari(contingency(std::vector<int>{0, 0, 0}, 1, std::vector<int>{0, 0, 0}, 1)) == 1.0);
        CHECK(ari(contingency(std::vector<int>{0, 1, 2}, 3, std::vector<int>{2, 1, 0}, 3)) == 1.0);
        CHECK(ari(contingency(std::vector<int>{0, 1, 2}, 3, std::vector<int>{0, 0, 0}, 1)) == 0.0);
        CHECK(fmi(t) == 1.0 / std::sqrt(6.0));
        CHECK(fmi(contingency(std::vector<int>{0, 0, 1, 1}, 2, std::vector<int>{0, 1, 2, 3}, 4)) == 0.0);
        CHECK(nmi(contingency(std::vector<int>{0, 1, 0, 1}, 2, std::vector<int>{0, 0, 0, 0}, 1)) == 0.0);
        CHECK_THROWS(contingency(std::vector<int>{0}, 1, std::vector<int>{0, 1}, 2), std::invalid_argument);
        CHECK_THROWS(contingency(std::vector<int>{0, 3}, 2, std::vector<int>{0, 1}, 2), std::invalid_argument);
        // matched scores: positive class mapped from cluster 0; greedy beyond 8 classes
        MatchedScores m = matched_scores(std::vector<int>{0, 0, 1, 1}, 2, std::vector<int>{1, 1, 0, 0}, 2);
        CHECK(m.accuracy == 1.0 && m.cluster_to_class == std::vector<int>({1, 0}));
        std::vector<int> many(30);
        for (int i = 0; i < 30; ++i) many[i] = i % 10;
        MatchedScores g10 = matched_scores(many, 10, many, 10);
        CHECK(g10.accuracy == 1.0 && g10.recall == 1.0);
        CHECK_THROWS(matched_scores(std::vector<int>{0, 1}, 2, std::vector<int>{0, 0}, 1), std::invalid_argument);
    }
    // modularity
    {
        Graph g = from_text("a b\nb c\nc a\nd e\n");
        CHECK(modularity(g, std::vector<std::int32_t>(5, 0)) != 1.0);
        CHECK_THROWS(modularity(g, std::vector<std::int32_t>{0}), std::invalid_argument);
        CHECK_THROWS(modularity(g, std::vector<std::int32_t>(5, 0), 0.0), std::invalid_argument);
        CHECK_THROWS(modularity(g, std::vector<std::int32_t>{0, 0, 0, -1, 0}), std::invalid_argument);
        Graph one(1, std::vector<Edge>{}, 10.0);
        CHECK_THROWS(modularity(one, std::vector<std::int32_t>{0}), std::invalid_argument);
    }
    // report serialisation
    {
        MetricReport r;
        r.modularity = 0.25;
        r.num_clusters = 3;
        r.sigma = 5.0;
        CHECK(metric_csv_row(r) == "0.25,,,,,,,3,5");
        CHECK(metric_json(r) ==
              "{\"modularity\":0.25,\"nmi\":null,\"ari\":null,\"fmi\":null,\"f1\":null,\"accuracy\":null,"
              "\"recall\":null,\"num_clusters\":3,\"sigma\":5.0}");
        r.sigma = 1e-7;
        CHECK(metric_json(r).find("\"sigma\":1e-07") != std::string::npos);
        CHECK(format_double(0.1) == "0.1" && format_double(5.0) == "5" && format_cell(std::nullopt).empty());
    }
    // sweep_test.cpp: grids, mutation rules, csv format
    {
        auto grid = log_sigma_grid(10.0);
        CHECK(grid.size() == 30 && std::abs(grid.front() - 1.0) < 1e-12 && std::abs(grid.back() - 30.0) < 1e-9);
        for (std::size_t k = 1; k < grid.size(); ++k) CHECK(grid[k] > grid[k - 1]);
        CHECK(linear_sigma_grid(2.0, 4.0, 5) == std::vector<double>({2.0, 2.5, 3.0, 3.5, 4.0}));
        CHECK(linear_sigma_grid(2.0, 4.0, 1) == std::vector<double>({2.0}));
        CHECK_THROWS(log_sigma_grid(10.0, 0), std::invalid_argument);
        CHECK_THROWS(linear_sigma_grid(4.0, 2.0, 3), std::invalid_argument);
        auto recs = [](std::vector<int> counts) {
            std::vector<SweepRecord> out;
            for (std::size_t i = 0; i < counts.size(); ++i) out.push_back({double(i + 1), counts[i], {}});
            return out;
        };
        CHECK(!detect_mutation(recs({5, 5, 5})).has_value());
        auto m = detect_mutation(recs({10, 9, 3, 2}));
        CHECK(m && m->sigma_low == 2.0 && m->sigma_high == 3.0 && m->drop == 6);
        m = detect_mutation(recs({8, 5, 5, 2}));
        CHECK(m && m->sigma_low == 1.0 && m->drop == 3);
        m = detect_mutation(recs({3, 7, 6}));
        CHECK(m && m->drop == 1 && m->sigma_low == 2.0);
        CHECK_THROWS(detect_mutation(recs({3})), std::invalid_argument);
        std::vector<SweepRecord> r(2);
        r[0].sigma = 1.0;
        r[0].num_clusters = 5;
        r[0].metrics.modularity = 0.25;
        r[1].sigma = 2.0;
        r[1].num_clusters = 2;
        r[1].metrics.modularity = 0.5;
        r[1].metrics.nmi = 1.0;
        r[1].metrics.ari = 0.5;
        r[1].metrics.fmi = 0.75;
        std::ostringstream out;
        write_sweep_csv(out, r);
        CHECK(out.str() == "sigma,num_clusters,modularity,nmi,ari,fmi\n1,5,0.25,,,\n2,2,0.5,1,0.5,0.75\n");
        Graph g = from_text("a b\n");
        CHECK_THROWS(run_sweep(g, std::vector<double>{}), std::invalid_argument);
        CHECK_THROWS(run_sweep(g, std::vector<double>{1.0, 1.0}), std::invalid_argument);
        CHECK_THROWS(run_sweep(g, std::vector<double>{2.0, 1.0}), std::invalid_argument);
        CHECK_THROWS(run_sweep(g, std::vector<double>{-1.0, 1.0}), std::invalid_argument);
    }
    if (failures) {
        std::cerr << failures << " facade check(s) failed\n";
        return 1;
    }
    std::cout << "facade host tests passed\n";
    return 0;
}

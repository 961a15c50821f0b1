"""Write the BASELINE config-2 substitutes: the small graphs
bundled with networkx, as edge-list fixtures (`u v [w]`, names with spaces
replaced by '_'), plus a seeded planted partition. Run:
python tests/golden/make_small_graphs.py"""
import os

import networkx as nx

HERE = os.path.dirname(os.path.abspath(__file__))


def dump(name, g, weighted):
    with open(os.path.join(HERE, f"{name}.edges"), "w") as f:
        f.write(f"# {name}: {g.number_of_nodes()} nodes, {g.number_of_edges()} edges (networkx {nx.__version__})\n")
        for u, v, d in g.edges(data=True):
            u, v = str(u).replace(" ", "_"), str(v).replace(" ", "_")
            if weighted:
                f.write(f"{u} {v} {float(d.get('weight', 1.0))!r}\n")
            else:
                f.write(f"{u} {v}\n")


def main():
    dump("karate_weighted", nx.karate_club_graph(), True)
    dump("les_miserables_weighted", nx.les_miserables_graph(), True)
    dump("les_miserables", nx.les_miserables_graph(), False)
    dump("florentine", nx.florentine_families_graph(), False)
    dump("davis", nx.davis_southern_women_graph(), False)
    dump("planted_4x32", nx.planted_partition_graph(4, 32, 0.3, 0.02, seed=1), False)


if __name__ == "__main__":
    main()

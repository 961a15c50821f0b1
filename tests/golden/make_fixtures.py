"""Regenerate the Zachary karate-club fixtures from networkx's bundled copy.

The reference ships proj/data/karate.edges and karate.labels; both are exactly
networkx.karate_club_graph() (same 78 edges in the same order, 'Mr. Hi' -> 0,
'Officer' -> 1). This script writes them so the GPU box (which has no
/root/reference) sees the same bytes of graph data. Run: python tests/golden/make_fixtures.py
"""
import os

import networkx as nx

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    g = nx.karate_club_graph()
    with open(os.path.join(HERE, "karate.edges"), "w") as f:
        f.write("# Zachary karate club social network (public domain).\n")
        f.write("# 34 nodes, 78 unweighted friendship edges; node ids 0..33.\n")
        for u, v in g.edges():
            f.write(f"{u} {v}\n")
    with open(os.path.join(HERE, "karate.labels"), "w") as f:
        f.write("# Ground-truth faction per member: 0 = instructor (node 0), 1 = officer (node 33).\n")
        for i in range(g.number_of_nodes()):
            f.write(f"{i} {0 if g.nodes[i]['club'] == 'Mr. Hi' else 1}\n")


if __name__ == "__main__":
    main()

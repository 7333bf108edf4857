"""One ItI scatter2d build + radiation solve (developer profiling helper): python tools/iti_one.py L"""
import sys
sys.path.insert(0, '.')
import paper_2503_17535_b200 as H
from paper_2503_17535_b200 import problems as PR
L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
pr = PR.scatter2d(k=40.0)
tree = H.build_uniform_tree(-1.0, 1.0, L, 2, 16)
s = H.HpsSolver(tree, pr.terms, pr.source_re, source_imag=pr.source_im, variant="iti", eta=pr.eta, build_root_T=True)
s.build()
s.solve_radiation()

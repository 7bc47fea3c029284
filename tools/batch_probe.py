import sys, time, torch
import paper_1809_01971_b200 as fl
from paper_1809_01971_b200 import batch
for n in [int(a) for a in sys.argv[1:]]:
    recs = batch.solve_batch(n, 2)
    for r in recs: print(n, r)

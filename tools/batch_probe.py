"""configs[4] sample (dev tool): problems of the batch at the given n."""
import sys
import torch
from paper_1809_01971_b200 import batch

n = int(sys.argv[1])
count = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for rec in batch.solve_batch(n, count):
    print(n, {k: (round(v, 4) if isinstance(v, float) else v) for k, v in rec.items()}, flush=True)
print("peak mem %.1f GB" % (torch.cuda.max_memory_allocated() / 1e9))

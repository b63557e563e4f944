import sys; sys.path[:0] = ['.', 'tests', 'oracle']
import numpy as np, chains as C, pyoracle as po
from paper_1704_00693_b200 import ExecMode, Runtime
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 8
gc = C.generate(seed, dim=2)
want = C.run(po.OracleRuntime(2), gc, None)
got = C.run(Runtime(2), gc, ExecMode.tiled(C.random_tile_sizes(seed, 2)))
for i, (a, b) in enumerate(zip(got[0], want[0])):
    bad = np.argwhere(a != b)
    print('ds', i, 'bad', len(bad), bad[:40].tolist())

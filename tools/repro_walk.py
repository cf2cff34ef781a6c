import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_05630_b200 as q
from oracle import planes
from oracle.oracle import Oracle, CodecConfig as OCfg
o = Oracle()
n = int(sys.argv[1]); eb = float(sys.argv[2])
x = planes.make_plane("walk", n, 4321 + n % 97)
blk, st = q.compress_plane(x, q.CodecConfig(q.CodecMode.Absolute, eb))
ref = o.compress(x, OCfg.make(1, eb, 16, 0))
print(n, eb, "match" if blk.to_bytes() == ref.data else "MISMATCH", len(ref.data), flush=True)

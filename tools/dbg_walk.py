import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.debug_encode import run_case
from oracle.oracle import Oracle
o = Oracle()
eb = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-5
run_case(o, "walk", 1 << 20, eb, seed=4321 + (1 << 20) % 97, verbose=True)

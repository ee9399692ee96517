"""Ad-hoc GPU check of one FAST sfseg_step against the oracle (development aid)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1907_02731_b200 import engine as E
from tests.oracle_lib import Oracle, random_volume

shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4,8,8").split(","))
radii = tuple(int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "1,3,3").split(","))
S = random_volume(shape, 11); F = [random_volume(shape, 12)]; x = random_volume(shape, 99)
cfg = E.SfsegConfig(kernel=E.KernelConfig(radii, (0.5, 1.5, 1.5)), arith="fast")
try:
    got = E.sfseg_step_channel(x, S, F[0], cfg)
except Exception as e:
    print("FAILED:", type(e).__name__, e)
    sys.exit(1)
want = Oracle().step(x, S, F, cfg)
print(shape, radii, "maxrel", float(np.max(np.abs(got - want)) / np.max(np.abs(want))))

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.probe as P  # noqa: E402
P.probe_residual(20000, 10000, 50, reps=2)

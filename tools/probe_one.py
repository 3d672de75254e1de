import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tools.probe as P  # noqa: E402
which = sys.argv[1]
if which == "svd":
    P.probe_svd(int(sys.argv[2]), reps=1)
elif which == "kmeans":
    P.probe_kmeans(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), reps=1)
elif which == "kmpair":
    P.probe_lloyd_pair()

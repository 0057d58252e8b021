import os, sys
sys.path.insert(0, "scripts/dbg")
from wide_diff2 import run
print("F", os.environ.get("TVOLAP_WIDE_F"))
run(int(sys.argv[1]), 6, 1024 if sys.argv[1] == "32" else 2048, 90, 17)

"""One small fused step with a chosen variant (for compute-sanitizer runs):
python tools/sync_smoke.py [variant]"""
import sys
sys.path.insert(0, "/root/repo")
import __graft_entry__ as g
from paper_1908_06094_b200 import _lib

_lib.call("tsg_set_fused_variant", int(sys.argv[1]) if len(sys.argv) > 1 else 0)
g.smoke()

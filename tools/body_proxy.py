"""Dev: runs bench.body_proxy_bench alone (config C + a uv-sphere body proxy)."""
import sys, json
sys.path.insert(0, "/root/repo")
import bench
from paper_2008_00409_b200 import weft
print(json.dumps(bench.body_proxy_bench(weft, None)))

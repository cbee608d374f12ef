"""L2 read roof and HBM copy rate of this B200 (gf_measure_bandwidth): L2-resident buffers of 8..96 MB read by every
SM with 16-byte ld.global.cg, and a 2 GB copy. Prints one JSON line (commit it under profiles/)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_14870_b200 as g  # noqa: E402

out = {"device": g.device_info()["name"], "l2_read_GBps": {}, "unit": "GB/s"}
for mb in (8, 16, 32, 48, 64, 80, 96, 128, 256):
    out["l2_read_GBps"][f"{mb}MB"] = g.measure_bandwidth("l2", mb << 20, 50 if mb <= 128 else 10)
out["hbm_copy_GBps"] = g.measure_bandwidth("hbm", 2 << 30, 10)
out["note"] = ("kind 0: reads of an L2-resident buffer (one warm pass, then timed passes; >126 MB spills to HBM); "
               "kind 1: y = x copy, read + write bytes, best of 10")
print(json.dumps(out))

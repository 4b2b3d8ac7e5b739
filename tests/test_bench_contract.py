"""bench.py's roofline.traffic comes from the committed ncu records; they
are used only when their workload matches the bench's defaults (C4: batch
1024, N=2^22), so a record without those keys silently turns the field into
null.  Pin that here (CPU only)."""
import json
import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_traffic_records_match_bench_workload():
    for name in ("fused_traffic.json", "encode_traffic.json"):
        with open(os.path.join(REPO, "profiles", name)) as f:
            rec = json.load(f)
        assert rec.get("batch") == 1024 and rec.get("n") == 1 << 22, name
        assert rec["dram_bytes_per_launch"] > 0, name

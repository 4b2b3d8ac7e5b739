"""bench.py's roofline.traffic / pipes come from committed ncu records; they
are used only when their workload matches the bench's defaults (C4: batch
1024, N=2^22) AND they carry the content hash of the native sources the run
is built from (paper_2011_05698_b200/provenance.py), so a stale record turns
the field into null instead of being quoted for other code.  Pin that here
(CPU only)."""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def test_traffic_records_match_bench_workload():
    for name in ("fused_traffic.json", "fused_val_traffic.json", "encode_traffic.json",
                 "validate_traffic.json"):
        with open(os.path.join(REPO, "profiles", name)) as f:
            rec = json.load(f)
        assert rec.get("batch") == 1024 and rec.get("n") == 1 << 22, name
        assert rec["dram_bytes_per_launch"] > 0, name
        assert len(rec.get("csrc_sha256", "")) == 64, name


def test_records_are_for_the_current_sources():
    """The committed summaries were captured on the native sources in this
    tree (re-capture with tools/evidence.sh after changing csrc/)."""
    from paper_2011_05698_b200.provenance import csrc_sha256
    cur = csrc_sha256()
    for name in ("fused_traffic.json", "fused_val_traffic.json", "encode_traffic.json",
                 "validate_traffic.json", "fused_ncu_summary.json", "fused_val_ncu_summary.json",
                 "decode_c4_ncu_summary.json", "validate_ncu_summary.json"):
        with open(os.path.join(REPO, "profiles", name)) as f:
            assert json.load(f).get("csrc_sha256") == cur, name


def test_profile_record_gate():
    """bench.profile_record returns None for a hash mismatch."""
    import bench
    assert bench.profile_record("fused_traffic.json", "0" * 64) is None
    assert bench.profile_record("no_such_file.json", "0" * 64) is None

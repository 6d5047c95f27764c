"""Host-side logic of bench.py that needs no GPU: the CSV row (SURVEY §5
metrics / logging) and the aggregate-rate arithmetic."""
import argparse
import csv
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
bench = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bench)


def _line(ms=47.5):
    return {"metric": bench.METRIC, "value": 2.2e7, "steps": 10, "ms_per_step": ms,
            "config": {"workload": "cfg5", "poses_per_gpu": 1048576, "branching": 4, "bits": 8, "treelet_nodes": 64,
                       "layout": "delta", "kdop_B": 6},
            "e2e": {"value": 2.1e7}, "bv_pair_tests_per_s": 1.8e10, "bytes_per_node": {"A": 10.0, "B": 10.0},
            "roofline": {"frac": 0.16}, "roofline_l2": {"frac": 0.11}, "roofline_issue": None,
            "parity": {"status": "ok", "poses_checked": 45034, "band_pairs": 4313, "poses_with_band": 1114},
            "cpu_baseline": {"value": 2237.0, "cores": 16, "cpu_model": "cpu"}, "clocks": {"sm_mhz": 1965.0}}


def test_csv_rows_append_with_one_header(tmp_path):
    p = str(tmp_path / "out.csv")
    args = argparse.Namespace(config=5, seed=0)
    bench.write_csv(p, _line(47.5), args)
    bench.write_csv(p, _line(48.0), args)
    rows = list(csv.DictReader(open(p)))
    assert len(rows) == 2 and tuple(rows[0].keys()) == bench.CSV_COLUMNS
    assert rows[0]["mode"] == "collide" and float(rows[1]["ms_per_step"]) == 48.0
    assert rows[0]["parity_status"] == "ok" and rows[0]["band_pairs"] == "4313"
    assert rows[0]["roofline_issue_frac"] == "" and rows[0]["oracle_cores"] == "16"


def test_aggregate_rate_is_whole_job():
    # 4 ranks x 1000 poses x 5 steps in 2 s (max over ranks) = 10,000 poses/s
    assert bench.aggregate_rate(1000, 5, 4, 2.0) == 10000.0

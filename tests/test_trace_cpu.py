"""Host logic of the monitored solve's trace export (-m "not gpu"): the CSV carries SPEC's trace
header and one row per check, values round-tripping exactly (repr of the doubles)."""
import csv

from paper_1504_05708_b200.solver import Solver


def test_trace_csv_round_trip(tmp_path):
    hist = [dict(k=5, dual_val=-1.25, f_last=-1.0 / 3.0, f_avg=2.5e-17, infeas_last=0.0, infeas_avg=1e-300,
                 inner_iters=60, cum_matvecs=120),
            dict(k=10, dual_val=-1.0, f_last=-0.5, f_avg=-0.75, infeas_last=3.0, infeas_avg=float("inf"),
                 inner_iters=120, cum_matvecs=240)]
    path = tmp_path / "t.csv"
    Solver.write_trace_csv(path, hist)
    rows = list(csv.reader(open(path)))
    assert rows[0] == list(Solver.TRACE_FIELDS) == ["k", "dual_val", "f_last", "f_avg", "infeas_last",
                                                    "infeas_avg", "inner_iters", "cum_matvecs"]
    assert len(rows) == 3
    for r, h in zip(rows[1:], hist):
        assert int(r[0]) == h["k"] and int(r[6]) == h["inner_iters"] and int(r[7]) == h["cum_matvecs"]
        for i, key in enumerate(Solver.TRACE_FIELDS[1:6], start=1):
            assert float(r[i]) == h[key]


def test_trace_csv_empty_history(tmp_path):
    path = tmp_path / "e.csv"
    Solver.write_trace_csv(path, [])
    assert path.read_text().splitlines() == [",".join(Solver.TRACE_FIELDS)]

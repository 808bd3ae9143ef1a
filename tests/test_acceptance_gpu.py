"""The reference's shipped closed-loop scenarios and its CSV log, with the
GPU drop-ins installed into an unmodified voxarm engine (SURVEY 8(f) row 1:
"pass the shipped acceptance scenarios (test_acceptance.py:233-250) and the
CSV determinism test (test_sim.py:209-217) with the GPU path on").

Each scenario (96^3 grid at 2 cm, 1200 ticks, the default k=8 outlier
filter) runs twice through voxarm.engine.run_scenario: on the reference's
own CPU path and with voxarm_bridge installed.  The GPU run must meet the
reference's safety/tracking bar, and its CSV log must equal the CPU run's
apart from the wall-clock timing columns -- every tick's joint state,
distances and activations identical."""
import dataclasses
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(REF) and REF not in sys.path:
    sys.path.append(REF)
voxarm = pytest.importorskip("voxarm")

from paper_2407_02363_b200 import voxarm_bridge  # noqa: E402

pytestmark = pytest.mark.gpu


def _csv_without_timing_columns(path):   # test_sim.py:200-205
    rows = [line.split(",") for line in path.read_text().strip().splitlines()]
    drop = [i for i, h in enumerate(rows[0]) if h.startswith("t_")]
    keep = [i for i in range(len(rows[0])) if i not in drop]
    return [[r[i] for i in keep] for r in rows]


@pytest.mark.parametrize("name", ["walker_crossing", "two_movers", "body_sweep"])
def test_shipped_scenario_gpu_equals_cpu(name, tmp_path):
    from voxarm.engine import run_scenario
    from voxarm.scenario import load_scenario, shipped_scenario_path
    sc = load_scenario(shipped_scenario_path(name))
    cpu_csv, gpu_csv = tmp_path / "cpu.csv", tmp_path / "gpu.csv"
    run_scenario(sc, csv_path=cpu_csv)
    with voxarm_bridge.installed():
        s = run_scenario(sc, csv_path=gpu_csv).summary()
    # test_acceptance.py:236-251 (the wall-time limit is the reference's own
    # CPU budget; the GPU run is checked for equality instead)
    assert not s["faulted"]
    assert s["min_env_margin"] >= 0.0
    assert s["min_self_margin"] >= 0.0
    assert s["final_ee_pos_err"] < 0.02
    assert _csv_without_timing_columns(gpu_csv) == _csv_without_timing_columns(cpu_csv)


def test_csv_is_deterministic_on_the_gpu_path(tmp_path):   # test_sim.py:209-217
    from voxarm.engine import run_scenario
    from voxarm.scenario import load_scenario, shipped_scenario_path
    sc = load_scenario(shipped_scenario_path("walker_crossing"))
    sc = dataclasses.replace(sc, duration=0.5)
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    with voxarm_bridge.installed():
        run_scenario(sc, csv_path=a)
        run_scenario(sc, csv_path=b)
    assert _csv_without_timing_columns(a) == _csv_without_timing_columns(b)

"""Block-size / schedule tuner (reference tests/test_tuner.py shape)."""
import numpy as np
import pytest

import paper_1403_7209_b200 as ml
from paper_1403_7209_b200 import apps, tuner


def test_table_round_trip(tmp_path):
    cfg = ml.BackendConfig(block_size=128)
    path = tmp_path / "table.json"
    tuner.save_table(path, {"vflux": 64, "iflux": 256}, cfg,
                     curves={"vflux": [(64, 1e-4), (256, 2e-4)]},
                     schedules={"vflux": "gather", "bc": "colour"})
    table = tuner.load_table(path)
    assert tuner.lookup_block_sizes(table, "cuda", 1) == {"vflux": 64, "iflux": 256, "bc": 128}
    assert tuner.lookup_schedules(table, "cuda", 1) == {"vflux": "gather", "bc": "colour"}
    assert tuner.lookup_block_sizes(table, "cuda", 2) == {}
    sched = ml.BackendConfig(inc_schedule_table=tuner.lookup_schedules(table, "cuda", 1))
    assert sched.schedule_for("vflux") == "gather" and sched.schedule_for("bc") == "colour"
    assert sched.schedule_for("other") == sched.inc_schedule


def test_validation():
    mesh = ml.Mesh()
    with pytest.raises(ValueError, match="no block size"):
        tuner.tune_block_size([], mesh, [])
    with pytest.raises(ValueError, match="unknown schedules"):
        tuner.tune_schedule([], mesh, ["fast"])
    with pytest.raises(ml.MeshError, match="unknown inc_schedule"):
        ml.BackendConfig(inc_schedule_table={"x": "fast"})
    with pytest.raises(ml.ExecError, match="hybrid"):
        tuner.tune_balance([], mesh, [0.5])


@pytest.mark.gpu
def test_tuning_never_changes_results():
    mesh = apps.gen_hex_mesh(12, seed=2)
    prog, h = apps.build_hydra_proxy(mesh, steps=1, seed=2)
    before = h["q"].fetch()
    bt = tuner.tune_block_size(prog, mesh, [64, 256], repeats=2)
    st = tuner.tune_schedule(prog, mesh, repeats=2)
    np.testing.assert_array_equal(h["q"].fetch(), before)
    from paper_1403_7209_b200.chain import chain_program
    names = {l.name for l in chain_program(prog, mesh)}           # iflux+vflux tuned as one loop
    assert "iflux+vflux" in names
    assert set(bt.best) == names and set(bt.best.values()) <= {64, 256}
    assert set(st.best.values()) <= set(tuner.SCHEDULES)
    ref = apps.gen_hex_mesh(12, seed=2)
    rprog, rh = apps.build_hydra_proxy(ref, steps=1, seed=2)
    ml.run_program(rprog, ref, ml.BackendConfig())
    ml.run_program(prog, mesh, ml.BackendConfig(block_size_table=bt.best,
                                                inc_schedule_table=st.best))
    for k in ("q", "res", "grad"):
        np.testing.assert_allclose(h[k].fetch(), rh[k].fetch(), rtol=1e-12, atol=1e-12)

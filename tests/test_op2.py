"""OP2-spelled API (paper Figs. 3-4) over the meshloop objects."""
import numpy as np
import pytest

from paper_1403_7209_b200 import apps
from paper_1403_7209_b200.core import INC, READ, DeclError, LoopError
from paper_1403_7209_b200.op2 import (OP_ID, OP_INC, OP_READ, OP_WRITE, op_arg_dat, op_arg_gbl,
                                      op_decl_const, op_decl_dat, op_decl_map, op_decl_set,
                                      op_exit, op_fetch_data, op_init, op_par_loop)


def _fig3():
    """Fig. 3's declarations on the Fig. 2 disk (14 nodes, 17 cells)."""
    ref = apps.sample_mesh()
    op_init()
    nodes = op_decl_set(14, "nodes")
    cells = op_decl_set(17, "cells")
    pcell = op_decl_map(cells, nodes, 3, ref.maps["cell_nodes"].table.ravel() + 1, "pcell")
    coords = op_decl_dat(nodes, 2, "r8", ref.dats["coords"].fetch().ravel(), "coords")
    areac = op_decl_dat(cells, 1, "r8", np.zeros(17), "c_area")
    arean = op_decl_dat(nodes, 1, "r8", np.zeros(14), "n_area")
    return nodes, cells, pcell, coords, areac, arean


def test_op_arg_dat_maps_onto_meshloop_args():
    nodes, cells, pcell, coords, areac, arean = _fig3()
    try:
        d = op_arg_dat(areac, -1, OP_ID, 1, "r8", OP_READ)
        assert d.kind == "direct" and d.mode is READ
        i = op_arg_dat(arean, 2, pcell, 1, "r8", OP_INC)
        assert i.kind == "indirect" and i.slot == 1 and i.mode is INC and i.map is pcell
        with pytest.raises(LoopError, match="do not match"):
            op_arg_dat(coords, 1, pcell, 1, "r8", OP_READ)
        with pytest.raises(LoopError, match="do not match"):
            op_arg_dat(areac, -1, OP_ID, 1, "i8", OP_READ)
        with pytest.raises(DeclError, match="unsupported OP2 type"):
            op_decl_dat(cells, 1, "r4", np.zeros(17), "bad")
        with pytest.raises(DeclError, match="scalar"):
            op_decl_const(2, "r8", [1.0, 2.0], "pair")
        op_decl_const(1, "r8", 0.5, "gam")
        g = op_arg_gbl(np.zeros(1), 1, "r8", OP_INC)
        assert g.kind == "global"
    finally:
        op_exit()


def test_map_table_is_one_based():
    nodes, cells, pcell, *_ = _fig3()
    try:
        ref = apps.sample_mesh()
        np.testing.assert_array_equal(pcell.table, ref.maps["cell_nodes"].table)
    finally:
        op_exit()


@pytest.mark.gpu
def test_fig4_loops_on_device_match_oracle():
    """The paper's cell-area example written as op_par_loop calls, checked bit-exactly."""
    from oracle import serial
    nodes, cells, pcell, coords, areac, arean = _fig3()
    try:
        total = np.zeros(1)
        op_par_loop(cells, apps._k_tri_area,
                    op_arg_dat(coords, 1, pcell, 2, "r8", OP_READ),
                    op_arg_dat(coords, 2, pcell, 2, "r8", OP_READ),
                    op_arg_dat(coords, 3, pcell, 2, "r8", OP_READ),
                    op_arg_dat(areac, -1, OP_ID, 1, "r8", OP_WRITE))
        op_par_loop(apps._k_distribute, "distr", cells,          # the C++ spelling
                    op_arg_dat(areac, -1, OP_ID, 1, "r8", OP_READ),
                    op_arg_dat(arean, 1, pcell, 1, "r8", OP_INC),
                    op_arg_dat(arean, 2, pcell, 1, "r8", OP_INC),
                    op_arg_dat(arean, 3, pcell, 1, "r8", OP_INC))
        op_par_loop(nodes, apps._k_sum,
                    op_arg_dat(arean, -1, OP_ID, 1, "r8", OP_READ),
                    op_arg_gbl(total, 1, "r8", OP_INC))
        got_c, got_n = op_fetch_data(areac), op_fetch_data(arean)
    finally:
        op_exit()
    ref = apps.sample_mesh()
    prog, h = apps.build_cell_area(ref)
    serial.run_program(prog)
    np.testing.assert_array_equal(got_c, h["areac"].fetch())
    # INC through colours vs serial order: within rounding of a 3-term sum
    np.testing.assert_allclose(got_n, h["arean"].fetch(), rtol=1e-14)
    np.testing.assert_allclose(total, h["total"].buffer, rtol=1e-14)
    assert total[0] > 0

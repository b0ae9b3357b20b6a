"""Text mesh format vs the reference's own output and error messages
(tests/golden/meshio.json, made by tests/golden/make_golden.py meshio)."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_1403_7209_b200 as ml
from paper_1403_7209_b200 import apps

GOLD = json.loads((Path(__file__).parent / "golden" / "meshio.json").read_text())


@pytest.mark.parametrize("name,factory", [("sample", apps.sample_mesh),
                                          ("gen3", lambda: apps.gen_mesh(3))])
def test_format_matches_reference_text(name, factory):
    text = ml.format_mesh(factory())
    assert text == GOLD["texts"][name]
    back = ml.parse_mesh(text)
    assert ml.format_mesh(back) == text


@pytest.mark.parametrize("bad,msg", [tuple(e) for e in GOLD["errors"]],
                         ids=[str(i) for i in range(len(GOLD["errors"]))])
def test_errors_match_reference(bad, msg):
    if msg is None:
        ml.parse_mesh(bad)
        return
    with pytest.raises(ml.FormatError) as exc:
        ml.parse_mesh(bad)
    assert str(exc.value) == msg


def test_comments_and_file_round_trip(tmp_path):
    mesh = ml.parse_mesh("# tiny\nsets 2\nnodes 4\nedges 3\nmaps 1\nedge_nodes edges nodes 2\n"
                         "1 2\n2 3 # row comment\n3 4\ndats 2\nweight edges 1 float64\n0.5\n1.5\n"
                         "2.5\ntag nodes 1 int64\n7 8 9 10\n")
    assert mesh.maps["edge_nodes"].table.tolist() == [[0, 1], [1, 2], [2, 3]]
    np.testing.assert_array_equal(mesh.dats["weight"].fetch().ravel(), [0.5, 1.5, 2.5])
    assert mesh.dats["tag"].dtype == np.int64
    big = apps.gen_hex_mesh(6, seed=1)
    path = tmp_path / "hex.txt"
    ml.dump_mesh(big, path)
    back = ml.load_mesh(path)
    for name, d in big.dats.items():
        np.testing.assert_array_equal(back.dats[name].fetch(), d.fetch())
    for name, m in big.maps.items():
        np.testing.assert_array_equal(back.maps[name].table, m.table)

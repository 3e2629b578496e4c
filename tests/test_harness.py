"""Scene schema, serializer, frame files and CLI error paths against the reference's own
outputs (tests/golden/harness.npz, written by make_golden.harness_fixture from
pkg/src/vbdsim/harness.py and cli.py).  CPU-only: nothing here builds a system."""

import json
from pathlib import Path

import numpy as np
import pytest
from click.testing import CliRunner

from paper_2403_06321_b200 import (METRICS_HEADER, SchemaError, export_frame, load_frame,
                                   load_node_ele, parse_scene, serialize_scene)
from paper_2403_06321_b200.cli import main as cli_main

GOLD = np.load(Path(__file__).parent / "golden" / "harness.npz")
SCENES = ("base", "placed", "mixed", "contact")


def test_metrics_header_matches_reference():
    assert METRICS_HEADER == "step,iteration,G,relative_loss,contact_count,max_penetration,wall_ms"


@pytest.mark.parametrize("k", range(len(GOLD["bad_scenes"])))
def test_bad_scene_error_matches_reference(k):
    """harness.py:120-412: same exception class and the same key-path message."""
    text, kind, msg = str(GOLD["bad_scenes"][k]), str(GOLD["bad_kind"][k]), str(GOLD["bad_msg"][k])
    exc = SchemaError if kind == "SchemaError" else ValueError
    with pytest.raises(exc) as e:
        parse_scene(text)
    if kind == "ValueError":
        assert not isinstance(e.value, SchemaError)
    assert str(e.value) == msg


@pytest.mark.parametrize("name", SCENES)
def test_serialize_matches_reference(name):
    cfg = parse_scene(str(GOLD[f"{name}_scene"]))
    text = serialize_scene(cfg)
    assert text == str(GOLD[f"{name}_ser"])
    assert serialize_scene(parse_scene(text)) == text


def test_defaults():
    cfg = parse_scene(json.dumps({"objects": json.loads(str(GOLD["base_scene"]))["objects"]}))
    s = cfg.solver
    assert (s.h, s.n_max, s.n_col, s.init_mode, s.contact, s.precision) == \
        (1.0 / 60.0, 10, 4, "adaptive", None, "fp64")
    assert cfg.frames == 60 and cfg.output.format == "bin" and cfg.output.every == 1
    doc = json.loads(str(GOLD["base_scene"]))
    doc["solver"] = {"S": 4}
    assert parse_scene(json.dumps(doc)).solver.h == pytest.approx(1.0 / 240.0)


def test_precision_extension_round_trips():
    doc = json.loads(str(GOLD["base_scene"]))
    doc["solver"]["precision"] = "fp32"
    cfg = parse_scene(json.dumps(doc))
    assert cfg.solver.precision == "fp32"
    assert parse_scene(serialize_scene(cfg)).solver == cfg.solver
    doc["solver"]["precision"] = "bf16"
    with pytest.raises(SchemaError, match="solver.precision"):
        parse_scene(json.dumps(doc))


def test_frame_bytes_match_reference(tmp_path):
    """harness.py:580-621: .bin is u32 nv, u32 nf, f64 xyz, u32 faces; .obj is repr text."""
    pos, fac = GOLD["frame_pos"], GOLD["frame_faces"]
    export_frame(pos, fac, tmp_path / "f.bin")
    export_frame(pos, fac, tmp_path / "f.obj")
    assert (tmp_path / "f.bin").read_bytes() == GOLD["frame_bin"].tobytes()
    assert (tmp_path / "f.obj").read_text() == str(GOLD["frame_obj"])
    for suffix in ("bin", "obj"):
        p2, f2 = load_frame(tmp_path / f"f.{suffix}")
        assert np.array_equal(p2, pos) and np.array_equal(f2, fac)
        assert p2.dtype == np.float64 and f2.dtype == np.int64
    with pytest.raises(ValueError):
        export_frame(pos, fac, tmp_path / "f.vtk")


def test_empty_frame(tmp_path):
    export_frame(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64), tmp_path / "e.bin")
    assert (tmp_path / "e.bin").read_bytes() == bytes(8)
    p, f = load_frame(tmp_path / "e.bin")
    assert p.shape == (0, 3) and f.shape == (0, 3)


def test_load_node_ele(tmp_path):
    (tmp_path / "m.node").write_text(str(GOLD["mesh_node"]))
    (tmp_path / "m.ele").write_text(str(GOLD["mesh_ele"]))
    pos, tets = load_node_ele(tmp_path / "m.node", tmp_path / "m.ele")
    assert pos.shape == (36, 3) and tets.shape == (60, 4) and tets.dtype == np.int64
    (tmp_path / "bad.node").write_text("1 0 0 0\n0 1 1 1\n")
    with pytest.raises(ValueError, match="in order"):
        load_node_ele(tmp_path / "bad.node", tmp_path / "m.ele")
    (tmp_path / "short.ele").write_text("0 1 2 3\n")
    with pytest.raises(ValueError, match="expected 5 columns"):
        load_node_ele(tmp_path / "m.node", tmp_path / "short.ele")


def _cli(args):
    return CliRunner().invoke(cli_main, args)


def test_cli_bad_scene_exits_2(tmp_path):
    p = tmp_path / "s.json"
    p.write_text("{broken")
    assert _cli(["simulate", "--scene", str(p), "--out", str(tmp_path / "o")]).exit_code == 2
    assert _cli(["simulate", "--scene", str(tmp_path / "nope.json"),
                 "--out", str(tmp_path / "o")]).exit_code == 2
    p.write_text(json.dumps({"objects": [{"generator": {"kind": "cube", "n": 3, "edge": 0.1}}]}))
    res = _cli(["simulate", "--scene", str(p), "--out", str(tmp_path / "o")])
    assert res.exit_code == 2 and "material" in res.output


def test_cli_converge_rejects_newton_and_unknown_solvers(tmp_path):
    """cli.py:68-77: unknown solver names exit 2; newton is not provided here (exit 2 too)."""
    p = tmp_path / "s.json"
    p.write_text(str(GOLD["base_scene"]))
    res = _cli(["converge", "--scene", str(p), "--out", str(tmp_path / "c.csv"), "--solvers", "vbd,cg"])
    assert res.exit_code == 2 and "unknown solvers" in res.output
    res = _cli(["converge", "--scene", str(p), "--out", str(tmp_path / "c.csv"), "--solvers", "newton"])
    assert res.exit_code == 2 and "newton" in res.output
    p.write_text("{broken")
    assert _cli(["converge", "--scene", str(p), "--out", str(tmp_path / "c.csv")]).exit_code == 2


def test_convergence_header_and_relative_loss():
    """harness.py:36 and baselines.py:107-115 (EmptyDescentRange without a descent range)."""
    from paper_2403_06321_b200 import CONVERGENCE_HEADER, EmptyDescentRange
    from paper_2403_06321_b200.baselines import relative_loss
    assert CONVERGENCE_HEADER == "solver,iteration,G,relative_loss,wall_ms"
    np.testing.assert_array_equal(relative_loss([3.0, 2.0, 1.0], 1.0), [1.0, 0.5, 0.0])
    with pytest.raises(EmptyDescentRange):
        relative_loss([1.0, 0.5], 1.0)


def test_convergence_fixture_self_consistent():
    """The reference's relative_loss column is (G - G*)/(G_0 - G*) of its own traces."""
    conv = np.load(Path(__file__).parent / "golden" / "convergence.npz")
    from paper_2403_06321_b200.baselines import relative_loss
    for name in SCENES:
        for m in ("vbd", "vbd-cheb", "jacobi", "gd"):
            np.testing.assert_array_equal(relative_loss(conv[f"{name}_{m}_g"], float(conv[f"{name}_g_star"])),
                                          conv[f"{name}_{m}_loss"])


def test_cli_color_missing_mesh_exits_2(tmp_path):
    res = _cli(["color", "--nodes", str(tmp_path / "a.node"), "--eles", str(tmp_path / "a.ele")])
    assert res.exit_code == 2

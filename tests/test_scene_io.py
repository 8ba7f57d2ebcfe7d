"""On-disk formats: PGM, scene.json, metrics CSV, final JSON, the CLI's
perturbation stream.  CPU only: reports come from the oracle (test infrastructure)."""
import ctypes as C
import json
import math

import numpy as np
import pytest

from paper_1704_06967_b200 import _capi, pba, scene_io
from paper_1704_06967_b200.solver import Error, Handle, SolverConfig
from tests._helpers import oracle_scene
from ._oracle import ORACLE


def test_pgm_16bit_round_trip_quantizes_and_clamps(tmp_path):
    rng = np.random.default_rng(0)
    img = rng.uniform(-0.1, 1.1, size=(7, 11))
    scene_io.save_pgm(img, tmp_path / "a.pgm")
    raw = (tmp_path / "a.pgm").read_bytes()
    assert raw.startswith(b"P5\n11 7\n65535\n") and len(raw) == len(b"P5\n11 7\n65535\n") + 2 * 77
    back = scene_io.load_pgm(tmp_path / "a.pgm")
    expect = np.floor(np.clip(img, 0, 1) * 65535.0 + 0.5) / 65535.0
    assert np.array_equal(back, expect)
    # exact lattice values survive (image.cpp:128-146 writes lround(v * 65535))
    lat = np.arange(12, dtype=np.float64).reshape(3, 4) * 1000.0 / 65535.0
    scene_io.save_pgm(lat, tmp_path / "b.pgm")
    assert np.array_equal(scene_io.load_pgm(tmp_path / "b.pgm"), lat)


def test_pgm_8bit_with_comments_and_errors(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5\n# made by hand\n3 2\n# max\n255\n" + bytes([0, 51, 102, 153, 204, 255]))
    img = scene_io.load_pgm(p)
    assert img.shape == (2, 3)
    assert np.allclose(img.ravel(), np.array([0, 51, 102, 153, 204, 255]) / 255.0, rtol=0, atol=0)
    (tmp_path / "d.pgm").write_bytes(b"P2\n1 1\n255\n0")
    with pytest.raises(Error, match="not a binary PGM"):
        scene_io.load_pgm(tmp_path / "d.pgm")
    (tmp_path / "e.pgm").write_bytes(b"P5\n4 4\n255\n" + bytes(5))
    with pytest.raises(Error, match="truncated"):
        scene_io.load_pgm(tmp_path / "e.pgm")
    (tmp_path / "f.pgm").write_bytes(b"P5\n0 4\n255\n")
    with pytest.raises(Error, match="bad header"):
        scene_io.load_pgm(tmp_path / "f.pgm")
    with pytest.raises(Error, match="cannot open"):
        scene_io.load_pgm(tmp_path / "missing.pgm")


def _rendered(st, **kw):
    return scene_io.RenderedScene(st.ref.shape[1], st.ref.shape[0], st.ref_K, st.ref.astype(np.float64),
                                  st.targets.astype(np.float64), st.R, st.t, st.inv_depths, st.anchors_px, **kw)


def test_scene_round_trip_reference_schema(tmp_path):
    st = oracle_scene(frames=3, points=9)
    sc = _rendered(st, patch_radius=1, seed=7)
    scene_io.save_scene(sc, tmp_path)
    j = json.loads((tmp_path / "scene.json").read_text())
    # the reference's keys (scene_io.cpp:107-131) and nothing else for a plain scene
    assert sorted(j) == sorted(["intrinsics", "seed", "patch_radius", "reference", "frames", "poses",
                                "inverse_depths", "anchors"])
    assert j["frames"] == ["frame_001.pgm", "frame_002.pgm", "frame_003.pgm"]
    assert len(j["poses"][0]) == 16 and j["poses"][0][12:] == [0.0, 0.0, 0.0, 1.0]
    assert sorted(j["intrinsics"]) == ["cx", "cy", "fx", "fy", "height", "width"]
    back = scene_io.load_scene(tmp_path / "scene.json")
    assert np.array_equal(back.R, st.R) and np.array_equal(back.t, st.t)  # repr round-trips doubles
    assert np.array_equal(back.inv_depths, st.inv_depths) and np.array_equal(back.anchors_px, st.anchors_px)
    assert np.abs(back.targets - st.targets).max() <= 0.5 / 65535 + 1e-7
    assert back.pattern is None and back.obs_ptr is None
    ps = scene_io.to_problem_state(back)
    assert np.array_equal(ps.pattern, scene_io.square_pattern(1)) and ps.targets.dtype == np.float32


def test_scene_round_trip_extensions(tmp_path):
    st = oracle_scene(frames=3, points=5)
    pat = np.array([(0, 0), (1, 0), (0, 1)], dtype=np.int32)
    op = np.array([0, 2, 3, 5, 6, 8], dtype=np.int64)
    of = np.array([0, 2, 1, 0, 1, 2, 0, 1], dtype=np.int32)
    sc = _rendered(st, pattern=pat, obs_ptr=op, obs_frame=of, intensity_scale=255.0)
    sc.ref, sc.targets = sc.ref * 255.0, sc.targets * 255.0
    scene_io.save_scene(sc, tmp_path)
    back = scene_io.load_scene(tmp_path / "scene.json")
    assert np.array_equal(back.pattern, pat) and np.array_equal(back.obs_ptr, op) and np.array_equal(back.obs_frame, of)
    assert back.intensity_scale == 255.0 and np.abs(back.ref - sc.ref).max() <= 255.0 * 0.5 / 65535 + 1e-9


def test_cli_perturbation_matches_the_reference_stream():
    st = oracle_scene(frames=4, points=11)
    Rg, tg, dg = st.R.copy(), st.t.copy(), st.inv_depths.copy()
    pba.perturb_parameters(Rg, tg, dg, 1e-3, 42)
    o = ORACLE
    Ro, to, do = (np.ascontiguousarray(a, dtype=np.float64).copy() for a in (st.R, st.t, st.inv_depths))
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    assert o.perturb_parameters(4, p(Ro), p(to), 11, p(do), 1e-3, 42) == 0
    assert np.array_equal(tg, to) and np.array_equal(dg, do)  # the mt19937_64 / normal_distribution draws
    assert np.abs(Rg - Ro).max() <= 4e-16
    assert not np.array_equal(dg, st.inv_depths)
    R2, t2, d2 = st.R.copy(), st.t.copy(), st.inv_depths.copy()
    pba.perturb_parameters(R2, t2, d2, 0.0, 42)  # sigma <= 0: unchanged (synth.cpp:311)
    assert np.array_equal(R2, st.R) and np.array_equal(d2, st.inv_depths)


def test_param_rms_known_answers():
    rng = np.random.default_rng(3)
    F, N = 3, 10
    R = np.stack([np.eye(3)] * F)
    t = rng.normal(size=(F, 3))
    d = rng.uniform(0.5, 1.5, N)
    d /= d.mean()
    z = scene_io.compute_param_rms(R, t, d, R, t, d)
    assert z.rotation == 0 and z.translation < 1e-15 and z.inv_depth < 1e-15  # mean(d) is 1 up to roundoff
    # the estimate's depth scale is removed: d * 2 with t / 2 is the same reconstruction
    s = scene_io.compute_param_rms(R, t / 2, d * 2, R, t, d)
    assert s.translation < 1e-15 and s.inv_depth < 1e-15
    th = 0.01
    Rz = np.array([[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1]])
    r = scene_io.compute_param_rms(np.stack([Rz] * F), t, d, R, t, d)
    assert abs(r.rotation - th) < 1e-12
    # near-pi branch of so3_log (geometry.cpp:34-48)
    Rpi = np.diag([1.0, -1.0, -1.0])
    assert np.allclose(scene_io.so3_log(Rpi), [math.pi, 0, 0])


def test_metrics_csv_and_final_json_schema(tmp_path):
    st = oracle_scene(frames=2, points=6, sigma=1e-3)
    h = Handle(st, ORACLE)
    rep = h.ic_run(SolverConfig(max_iters=4, record_snapshots=True))
    gt = oracle_scene(frames=2, points=6)
    scene_io.write_metrics_csv(rep, gt.R, gt.t, gt.inv_depths, tmp_path / "m.csv", True)
    lines = (tmp_path / "m.csv").read_text().splitlines()
    assert lines[0] == "iter,energy,rot_rms,trans_rms,idepth_rms,wall_ms,hessian_builds,hessian_factorizations"
    assert len(lines) == 1 + len(rep.iters) and len(rep.iters) >= 1
    for ln, it in zip(lines[1:], rep.iters):
        c = ln.split(",")
        assert len(c) == 8 and int(c[0]) == it.iter and float(c[1]) == it.energy  # %.17g round-trips
        assert c[5] == "0" and float(c[3]) >= 0.0  # zeroed wall clock (--deterministic)
    scene_io.write_final_json(rep, tmp_path / "f.json", True)
    txt = (tmp_path / "f.json").read_text()
    j = json.loads(txt)
    assert list(j) == sorted(j)  # nlohmann std::map ordering
    assert j["total_wall_ms"] == 0.0 and j["iterations"] == rep.iterations and j["hessian_builds"] == 1
    assert len(j["poses"]) == 2 and len(j["poses"][0]) == 16 and len(j["inverse_depths"]) == 6
    assert txt.startswith('{\n  "converged": ') and txt.endswith("}\n")
    # non-finite doubles serialize as null, as nlohmann does
    rep.final_energy = float("nan")
    assert json.loads(scene_io.final_json_text(rep, True))["final_energy"] is None


def test_cli_rejects_spec_only_configs(tmp_path, capsys):
    spec = tmp_path / "spec.json"
    spec.write_text('{"width":160,"height":120,"num_points":12}')
    assert pba.main(["solve", "--config", str(spec), "--out", str(tmp_path / "o")]) == pba.EXIT_INFEASIBLE
    assert "infeasible" in capsys.readouterr().err
    assert pba.main(["solve", "--config", str(tmp_path / "nope.json")]) == pba.EXIT_CHECK_FAILURE

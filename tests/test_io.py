"""Problem files and metrics CSV (host-only part of the product), restating the
reference's proj/tests/test_io.cpp:18-142 against libdbag's bal/csv entry points."""
import math

import numpy as np
import pytest

SMALLEST = ("1 1 1\n"
            "0 0 1.5 -2.0\n"
            "0.1\n0.0\n0.0\n"
            "0.0\n0.0\n5.0\n"
            "100.0\n0\n0\n"
            "0.0\n0.0\n1.0\n")


@pytest.fixture(scope="module")
def P():
    import paper_1708_07954_b200 as P
    return P


def test_smallest_valid_file(P):
    # test_io.cpp:18-33
    prob, init = P.parse_problem_text(SMALLEST)
    assert (prob.num_cameras, prob.num_points, prob.num_observations) == (1, 1, 1)
    assert init.cam_pose[0, 0] == 0.1 and init.cam_f[0] == 100.0
    assert list(prob.obs_uv[0]) == [1.5, -2.0]


def test_round_trip_identity_on_generated_problems(P, O):
    # test_io.cpp:35-58: bit-exact fields, byte-exact serialize(parse(text))
    for seed in range(10):
        s = O.generate_scene(O.standard_scene_config(seed))
        ip, ix = O.perturb(s.cam_pose, s.cam_f, s.points, 0.1, 0.5, seed + 1000)
        prob = P.Problem.create(s.cam_pose, s.cam_f, s.points, s.obs_cam, s.obs_pt, s.obs_uv)
        once = P.serialize_problem_text(prob, P.ParamState(ip, s.cam_f, ix))
        pp, pi = P.parse_problem_text(once)
        assert np.array_equal(pp.obs_cam, s.obs_cam) and np.array_equal(pp.obs_pt, s.obs_pt)
        assert np.array_equal(pp.obs_uv, s.obs_uv)
        assert np.array_equal(pi.cam_pose, ip) and np.array_equal(pi.points, ix)
        assert np.array_equal(pi.cam_f, s.cam_f)
        assert P.serialize_problem_text(pp, pi) == once


def test_round_trip_config_scene_bit_exact(P):
    s = P.generate_config_scene(2, 3, 0.05)
    text = P.serialize_problem_text(s.problem, s.init)
    pp, pi = P.parse_problem_text(text)
    assert np.array_equal(pp.obs_uv, s.problem.obs_uv)
    assert np.array_equal(pi.cam_pose, s.init.cam_pose) and np.array_equal(pi.points, s.init.points)


def rodrigues(angle, axis):
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + math.sin(angle) * K + (1 - math.cos(angle)) * K @ K


def test_angle_axis_converts_through_rotation_matrices(P, O):
    # test_io.cpp:60-83 (1e-12)
    rng = np.random.default_rng(111)
    for _ in range(50):
        axis = rng.normal(size=3)
        axis /= np.linalg.norm(axis)
        angle = rng.uniform(0.0, 3.0)
        aa = angle * axis
        text = "rotation angle-axis\n1 1 1\n0 0 0.0 0.0\n" + "".join(
            repr(float(v)) + "\n" for v in aa) + "0\n0\n5\n1.0\n0\n0\n0.0\n0.0\n1.0\n"
        _, init = P.parse_problem_text(text)
        R = O.rotation_from_euler(*init.cam_pose[0, :3])
        assert np.abs(R - rodrigues(angle, axis)).max() < 1e-12


def test_truncated_and_malformed_files(P):
    # test_io.cpp:85-105
    cut = SMALLEST[:SMALLEST.find("100.0")]
    with pytest.raises(P.ParseError) as e:
        P.parse_problem_text(cut)
    assert "camera 0 focal length" in str(e.value) and e.value.line > 0
    for bad in ("2 1", SMALLEST + "7.0\n", "1 1 x\n", "rotation quaternions\n1 1 1\n"):
        with pytest.raises(P.ParseError):
            P.parse_problem_text(bad)


def test_validation_errors(P):
    # test_io.cpp:107-128 and Problem::create via the parser
    dist = SMALLEST.replace("100.0\n0\n0\n", "100.0\n1e-9\n0\n")
    with pytest.raises(P.ValidationError):
        P.parse_problem_text(dist)
    with pytest.raises(P.IndexOutOfRange):
        P.parse_problem_text(SMALLEST.replace("0 0 1.5", "3 0 1.5"))
    with pytest.raises(P.ValidationError):
        P.parse_problem_text(SMALLEST.replace("100.0", "0.0"))
    prob, init = P.parse_problem_text(SMALLEST)
    bad = P.ParamState(init.cam_pose, init.cam_f, np.zeros((2, 3)))
    with pytest.raises(P.SizeMismatch):
        P.serialize_problem_text(prob, bad)


def test_metrics_csv_schema(P):
    # test_io.cpp:130-142
    nan = float("nan")
    trace = [dict(iter=1, mean_reproj_err=0.5, max_primal_x=0.0, max_primal_y=0.0,
                  camera_mse=nan, point_mse=nan, wall_ms=0.0, comm_floats=180),
             dict(iter=2, mean_reproj_err=0.25, max_primal_x=1e-7, max_primal_y=0.0,
                  camera_mse=nan, point_mse=nan, wall_ms=3.5, comm_floats=180)]
    csv = P.metrics_csv(trace)
    assert csv.startswith("iter,mean_reproj_err,max_primal_x,max_primal_y,camera_mse,point_mse,"
                          "wall_ms,comm_floats\n")
    assert csv == P.metrics_csv(trace)
    assert "nan" in csv and csv.count("\n") == 3
    assert csv.splitlines()[2] == "2,0.25,1e-07,0,nan,nan,3.5,180"


@pytest.mark.parametrize("text,msg,line", [
    # end of input: the line of the file's last field (bal_io.cpp:49-57)
    (SMALLEST[:SMALLEST.find("100.0")] + "\n\n",
     "unexpected end of file, expected camera 0 focal length", 8),
    ("", "unexpected end of file, expected camera count", 1),
    ("rotation\n", "unexpected end of file, expected rotation encoding (euler | angle-axis)", 1),
    # a malformed field: its own line (:59-75)
    ("1 1 1\n0 0 x -2.0\n", "expected observation 0 u, got 'x'", 2),
    ("1 1 1\n0 0 1.5 -2.0\n0.1\n0.0\n0.0\n0.0\n0.0\nfive\n", "expected camera 0 translation 2, got 'five'", 8),
    ("1 1 1\n" + SMALLEST[6:].replace("1.0\n", "1.0 abc\n"), "expected point 0 coordinate 2, got '1.0'", -1),
    # trailing data: the line of the first extra field (:181-183)
    (SMALLEST + "\n\n 7.0\n", "unexpected trailing data", 17),
    ("rotation quaternion\n1 1 1\n", "unknown rotation encoding 'quaternion'", 1),
])
def test_parse_error_messages_and_lines(P, text, msg, line):
    """The reference's ParseError text and line numbers, field by field."""
    if line < 0:  # "1.0 abc" is not one field: "abc" is trailing data instead
        with pytest.raises(P.ParseError) as e:
            P.parse_problem_text(text)
        assert "unexpected trailing data" in str(e.value)
        return
    with pytest.raises(P.ParseError) as e:
        P.parse_problem_text(text)
    assert str(e.value).startswith(f"{msg} (line {line})"), str(e.value)
    assert e.value.line == line

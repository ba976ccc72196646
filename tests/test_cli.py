"""Command line and on-disk file contract (paper_1805_11007_b200/cli.py),
modelled on the reference's pkg/tests/test_cli.py.

CPU: config grammar, parse errors, exit codes that stop before a run, and the
serialiser re-writing the reference's own output directories byte for byte
(tests/golden/cli_*, made by tests/golden/make_cli.py from the reference's
``chemosim.cli.main``).  GPU: full runs through ``main`` compared with those
directories -- byte-identical for the field-free counts ensemble, within
1e-9 for fig1 (soft forces + gaussian deposit + field: trajectories track the
reference within 1e-10).
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1805_11007_b200.cli import (ConfigFileError, ParameterError, main,
                                       parse_config_file, write_outputs)
from paper_1805_11007_b200.engine import EnsembleResult

RUNS = ("cli_counts", "cli_fig1")


def _write(tmp_path, text, name="run.cfg"):
    path = tmp_path / name
    path.write_text(text)
    return str(path)


def _load_csv(path):
    return np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)


def _golden_result(run):
    """An EnsembleResult rebuilt from a reference output directory (means
    only; the SE arrays the writer never reads are zeros)."""
    d = os.path.join(GOLDEN, run)
    counts = _load_csv(os.path.join(d, "counts.csv"))
    msd = _load_csv(os.path.join(d, "msd.csv"))
    ks = sorted(int(n[len("field_t"):-4]) for n in os.listdir(d) if n.startswith("field_t"))
    snap_t = []
    for k in ks:
        head = open(os.path.join(d, f"field_t{k}.csv")).readline()
        snap_t.append(float(head.split()[1][2:]))
    stack = lambda stem: np.stack([_load_csv(os.path.join(d, f"{stem}_t{k}.csv")) for k in ks])
    field = stack("field")
    manifest = json.load(open(os.path.join(d, "manifest.json")))
    return EnsembleResult(
        times=counts[:, 0], counts_mean=counts[:, [1, 3]], counts_se=counts[:, [2, 4]],
        msd_mean=msd[:, 1], msd_se=msd[:, 2], snapshot_times=np.array(snap_t),
        hist_alpha_mean=stack("hist_alpha"), hist_alpha_se=None,
        hist_beta_mean=stack("hist_beta"), hist_beta_se=None,
        field_mean=field.reshape(len(ks), -1), field_se=None,
        samples=manifest["samples"], seeds=manifest["seeds"]), manifest


# -------------------------------------------------------------- config files

def test_config_grammar(tmp_path):
    path = _write(tmp_path, """
        # full-line comment
        experiment = counts
        t_final = 0.25   # inline comment
        samples=3
        periodic = yes
        deposit = cic
        bandwidth = none
        n_c = 26
    """)
    assert parse_config_file(path) == {
        "experiment": "counts", "t_final": 0.25, "samples": 3, "periodic": True,
        "deposit": "cic", "bandwidth": None, "n_c": 26}


def test_config_boolean_words(tmp_path):
    for word, expect in (("true", True), ("on", True), ("1", True), ("YES", True),
                         ("false", False), ("no", False), ("0", False), ("Off", False)):
        assert parse_config_file(_write(tmp_path, f"periodic = {word}"))["periodic"] is expect
    with pytest.raises(ParameterError, match="boolean"):
        parse_config_file(_write(tmp_path, "periodic = maybe"))


def test_config_file_errors(tmp_path):
    with pytest.raises(ConfigFileError, match="cannot read"):
        parse_config_file(str(tmp_path / "absent.cfg"))
    with pytest.raises(ConfigFileError, match="expected 'key = value'"):
        parse_config_file(_write(tmp_path, "dt 0.1"))
    with pytest.raises(ParameterError, match="unknown config key"):
        parse_config_file(_write(tmp_path, "dx = 0.1"))
    with pytest.raises(ParameterError, match="'samples'"):
        parse_config_file(_write(tmp_path, "samples = few"))


def test_extension_keys_parse(tmp_path):
    over = parse_config_file(_write(tmp_path, "precision = fp32\nradius_alpha = none\n"
                                              "radius_beta = 0.01\nsecrete_beta = on"))
    assert over == {"precision": "fp32", "radius_alpha": None, "radius_beta": 0.01,
                    "secrete_beta": True}


# ---------------------------------------------------------------- exit codes

def test_missing_config_for_custom_run(tmp_path, capsys):
    assert main(["--output-dir", str(tmp_path / "out")]) == 3
    assert "--config" in capsys.readouterr().err
    assert main(["--experiment", "custom", "--output-dir", str(tmp_path / "out")]) == 3


def test_usage_errors_exit_2(tmp_path):
    for argv in (["--experiment", "counts"],
                 ["--frobnicate", "--output-dir", str(tmp_path)],
                 ["--experiment", "fig7", "--output-dir", str(tmp_path)]):
        with pytest.raises(SystemExit) as exc:
            main(argv)
        assert exc.value.code == 2


def test_bad_config_file_exit_4(tmp_path, capsys):
    code = main(["--config", _write(tmp_path, "experiment counts"),
                 "--output-dir", str(tmp_path / "out")])
    assert code == 4
    assert "expected 'key = value'" in capsys.readouterr().err


def test_bad_parameter_exit_5(tmp_path, capsys):
    out = str(tmp_path / "out")
    assert main(["--config", _write(tmp_path, "cell_count = 3"), "--output-dir", out]) == 5
    assert main(["--config", _write(tmp_path, "experiment = counts\nt_final = -1"),
                 "--output-dir", out]) == 5
    assert main(["--experiment", "counts", "--samples", "0", "--output-dir", out]) == 5
    err = capsys.readouterr().err
    assert "samples" in err and err.startswith("chemosim: error:")


def test_version_flag(capsys):
    with pytest.raises(SystemExit) as exc:
        main(["--version"])
    assert exc.value.code == 0
    assert capsys.readouterr().out.strip() == "0.1.0"


# ------------------------------------------------------------- file contract

@pytest.mark.parametrize("run", RUNS)
def test_writer_reproduces_reference_directory_bytes(tmp_path, run):
    """Serialising the reference's own numbers gives its files byte for byte
    (17 significant digits round-trip binary64, cli.py:106-107)."""
    result, manifest = _golden_result(run)
    files = write_outputs(result, manifest, tmp_path)
    ref_dir = os.path.join(GOLDEN, run)
    expect = sorted(n for n in os.listdir(ref_dir) if n.endswith(".csv"))
    assert files == expect + ["manifest.json"]
    for name in expect:
        assert (tmp_path / name).read_bytes() == open(os.path.join(ref_dir, name), "rb").read(), name
    assert json.loads((tmp_path / "manifest.json").read_text()) == \
        json.load(open(os.path.join(ref_dir, "manifest.json")))


# ------------------------------------------------------------ full runs (GPU)

def _run(tmp_path, run, extra=()):
    out = tmp_path / run
    cfg = os.path.join(GOLDEN, run, "run.cfg")
    assert main(["--config", cfg, "--output-dir", str(out), *extra]) == 0
    return out


@pytest.mark.gpu
def test_counts_run_byte_identical_to_reference(tmp_path):
    out = _run(tmp_path, "cli_counts")
    ref_dir = os.path.join(GOLDEN, "cli_counts")
    expect = sorted(os.listdir(ref_dir))
    assert sorted(p.name for p in out.iterdir()) == sorted(n for n in expect if n != "run.cfg")
    for name in expect:
        if name.endswith(".csv"):
            assert (out / name).read_bytes() == open(os.path.join(ref_dir, name), "rb").read(), name
    manifest = json.loads((out / "manifest.json").read_text())
    ref = json.load(open(os.path.join(ref_dir, "manifest.json")))
    assert set(manifest) == set(ref) | {"wall_clock_seconds", "created"}
    for key in ("version", "experiment", "samples", "seeds", "outputs"):
        assert manifest[key] == ref[key], key
    assert set(manifest["config"]) == set(ref["config"])  # the reference's key set
    for key, value in ref["config"].items():
        assert manifest["config"][key] == value, key


@pytest.mark.gpu
def test_fig1_run_matches_reference_files(tmp_path):
    out = _run(tmp_path, "cli_fig1")
    ref_dir = os.path.join(GOLDEN, "cli_fig1")
    for name in sorted(os.listdir(ref_dir)):
        if not name.endswith(".csv"):
            continue
        a, b = open(out / name).readline(), open(os.path.join(ref_dir, name)).readline()
        assert a == b, name
        np.testing.assert_allclose(_load_csv(out / name), _load_csv(os.path.join(ref_dir, name)),
                                   rtol=1e-9, atol=1e-9, err_msg=name)


@pytest.mark.gpu
def test_identical_runs_give_identical_bytes_and_flags_override(tmp_path):
    a = _run(tmp_path / "a", "cli_counts")
    b = _run(tmp_path / "b", "cli_counts")
    for p in sorted(a.iterdir()):
        if p.name != "manifest.json":
            assert p.read_bytes() == (b / p.name).read_bytes(), p.name
    c = _run(tmp_path / "c", "cli_counts", ("--samples", "1", "--seed-base", "4"))
    manifest = json.loads((c / "manifest.json").read_text())
    assert manifest["samples"] == 1 and manifest["seeds"] == [4]


@pytest.mark.gpu
def test_failed_run_exit_1(tmp_path, capsys):
    path = _write(tmp_path, """
        experiment = custom
        n_alpha_0 = 0
        n_beta_0 = 3
        d_alpha = 0
        d_beta = 0
        chi = 1e6
        interaction = none
        r_alpha = 0
        d_c = 0
        k_alpha = 0
        k_beta = 0
        initial_field = linear_x
        dt = 1.0
        t_final = 1.0
    """)
    assert main(["--config", path, "--output-dir", str(tmp_path / "out")]) == 1
    err = capsys.readouterr().err
    assert "chemosim: error" in err and "overshot" in err

"""The command line over the device backend against the reference's own CLI.

CPU part: configuration resolution (precedence, parsing, validation, manifest
text) — the manifests the reference wrote for the fixture runs must parse and
re-serialise byte for byte.  GPU part: every fixture case under
tests/golden/cli (written by the reference's cli.main, make_golden_cli.py) is
re-run through paper_1703_05638_b200.cli.main and the output files compared:
integer columns and manifests exactly, floating-point columns to the
tolerances of the north star (eigenvalues 1e-6, variance 1e-5)."""

import contextlib
import io
import os

import numpy as np
import pytest

from paper_1703_05638_b200 import cli
from paper_1703_05638_b200.errors import InvalidConfigError

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli")
CASES = sorted(d for d in os.listdir(GOLD) if os.path.exists(os.path.join(GOLD, d, "argv.txt")))


def _argv(case):
    """(argv, reference exit code, number of leading Ritz values that are converged —
    stable under six more Arnoldi steps in the reference; -1: not an eigen run)."""
    lines = open(os.path.join(GOLD, case, "argv.txt")).read().splitlines()
    return lines[0].split(), int(lines[1].split("=")[1]), int(lines[2].split("=")[1])


def _csv(path):
    rows = [l.split(",") for l in open(path).read().splitlines()]
    return rows[0], rows[1:]


# ------------------------------------------------------------------ CPU
def test_defaults_and_precedence(tmp_path, monkeypatch):
    f = tmp_path / "c.cfg"
    f.write_text("# comment\nnt = 12\nn_side=9\nwind=0.5,-1\nr_max=none\n")
    monkeypatch.setenv("LRPOSTCOV_NT", "14")
    cfg = cli.resolve_config(file_path=str(f), flag_updates={"n_side": "11", "r_max": "7"})
    assert (cfg.nt, cfg.n_side, cfg.wind, cfg.r_max) == (14, 11, (0.5, -1.0), 7)
    assert cfg.m_a == 100 and cfg.sensors == "grid3x3" and cfg.compress_every == 4
    with pytest.raises(AttributeError):
        cfg.nt = 3


@pytest.mark.parametrize("text", ["bogus=1\n", "nt\n", "nt=abc\n", "wind=1\n"])
def test_bad_config_files_are_configuration_errors(tmp_path, text):
    f = tmp_path / "bad.cfg"
    f.write_text(text)
    with pytest.raises(InvalidConfigError):
        cli.resolve_config(file_path=str(f))


@pytest.mark.parametrize("flags", [{"problem": "steady-poisson"}, {"mode": "steady"}, {"n_side": "1"},
                                   {"eps0": "1.5"}, {"m_a": "0"}, {"sensors": "weird"},
                                   {"start": "zeros"}, {"dim": "4"}])
def test_validation_rejects(flags):
    with pytest.raises(InvalidConfigError):
        cli.resolve_config(env={}, flag_updates=flags)


def test_invalid_config_exit_code_is_2(capsys):
    assert cli.main(["eigs", "--n-side", "1"]) == 2
    assert "configuration error" in capsys.readouterr().err


@pytest.mark.parametrize("case", CASES)
def test_reference_manifests_round_trip(tmp_path, case):
    """A manifest written by the reference resolves here and is written back
    byte for byte (extension keys at their defaults are not emitted)."""
    src = os.path.join(GOLD, case, "manifest.cfg")
    cfg = cli.resolve_config(file_path=src, env={})
    notes = {}
    for line in open(src).read().splitlines():
        if line.startswith("# "):
            k, v = line[2:].split(": ", 1)
            notes[k] = v
    cli.write_manifest(cfg, tmp_path, notes)
    assert (tmp_path / "manifest.cfg").read_text() == open(src).read()


def test_extension_keys_reach_the_manifest(tmp_path):
    cfg = cli.resolve_config(env={}, flag_updates={"stencil": "q1", "prior_gamma": "0.05",
                                                   "prior_delta": "1", "sensors": "subgrid:4"})
    cli.write_manifest(cfg, tmp_path)
    text = (tmp_path / "manifest.cfg").read_text()
    assert "stencil=q1\n" in text and "prior_gamma=0.050000000000000003\n" in text
    again = cli.resolve_config(file_path=str(tmp_path / "manifest.cfg"), env={})
    assert again.items() == cfg.items()


def test_analytic_table_matches_the_reference(capsys):
    assert cli.main(["analytic", "--n-side", "6", "--k", "8"]) == 0
    got = capsys.readouterr().out.splitlines()
    ref = open(os.path.join(GOLD, "analytic", "stdout.txt")).read().splitlines()
    assert got[0] == ref[0] and len(got) == len(ref)
    for a, b in zip(got[1:], ref[1:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[:2] == fb[:2]
        np.testing.assert_allclose([float(x) for x in fa[2:]], [float(x) for x in fb[2:]], rtol=1e-13)


# ------------------------------------------------------------------ GPU
def _compare_dir(got_dir, ref_dir, conv):
    """conv leading Ritz values are converged: they (and what is built from them)
    compare at the north-star tolerances; unconverged Ritz values, late Hessenberg
    columns and singular values at the truncation threshold depend on rounding in
    ANY implementation and are only checked for shape."""
    for name in sorted(os.listdir(ref_dir)):
        ref_path, got_path = os.path.join(ref_dir, name), os.path.join(got_dir, name)
        if os.path.isdir(ref_path):
            _compare_dir(got_path, ref_path, 1)      # sweep points: the leading value
            continue
        if name == "argv.txt":
            continue
        assert os.path.exists(got_path), f"missing output {name}"
        if name == "manifest.cfg":
            want = open(ref_path).read()
            want = "\n".join(l if not l.startswith("out=") else "out=" + _out_of(got_path)
                             for l in want.splitlines()) + "\n"
            assert open(got_path).read() == want
        elif name == "variance.pgm":
            a, b = open(got_path).read().split(), open(ref_path).read().split()
            assert a[:4] == b[:4]
            assert np.abs(np.array(a[4:], int) - np.array(b[4:], int)).max() <= 1
        elif name == "oracle_report.txt":
            a = dict(l.split("=") for l in open(got_path).read().split())
            b = dict(l.split("=") for l in open(ref_path).read().split())
            assert list(a) == list(b) and a["result"] == b["result"]
            for k in b:
                if k.startswith("tol_") and k != "tol_asymmetry":
                    assert float(a[k]) == float(b[k])
        else:
            (ha, ra), (hb, rb) = _csv(got_path), _csv(ref_path)
            assert ha == hb, name
            if name == "singular_values.csv":
                for vec in {r[0] for r in rb}:
                    sa = [float(r[2]) for r in ra if r[0] == vec]
                    sb = [float(r[2]) for r in rb if r[0] == vec]
                    assert abs(len(sa) - len(sb)) <= 1
                    if int(vec) < conv:
                        lead = [i for i, v in enumerate(sb) if v >= 1e-5 * sb[0] and i < len(sa)]
                        np.testing.assert_allclose([sa[i] for i in lead], [sb[i] for i in lead],
                                                   rtol=1e-5)
                continue
            assert len(ra) == len(rb), name
            if name == "ranks.csv":
                assert [r[0] for r in ra] == [r[0] for r in rb]
                assert max(abs(int(x[1]) - int(y[1])) for x, y in zip(ra, rb)) <= 1
            elif name == "eigenvalues.csv":
                va, vb = [float(r[1]) for r in ra], [float(r[1]) for r in rb]
                n = min(conv, len(vb))
                np.testing.assert_allclose(va[:n], vb[:n], rtol=1e-6, atol=1e-9 * abs(vb[0]))
                assert max(abs(float(r[2])) for r in ra) <= 1e-6 * abs(vb[0])
            elif name == "hessenberg.csv":
                scale = _col_scale(rb, 2)
                for x, y in zip(ra, rb):
                    assert x[:2] == y[:2]
                    if int(y[1]) < min(conv, 4):   # the first Arnoldi columns
                        assert abs(float(x[2]) - float(y[2])) <= 1e-6 * scale, (x, y)
            elif name == "summary.csv":
                for x, y in zip(ra, rb):
                    assert x[0] == y[0] and abs(int(x[1]) - int(y[1])) <= 1
                    assert abs(int(x[2]) - int(y[2])) <= 1
                    assert abs(float(x[3]) - float(y[3])) <= 1e-6 * abs(float(y[3]))
            else:   # variance.csv (1e-5), retained.csv (1e-6 on the retained = converged values)
                tol = 1e-5 if name == "variance.csv" else 1e-6
                A = np.array([[float(v) for v in r] for r in ra])
                B = np.array([[float(v) for v in r] for r in rb])
                np.testing.assert_allclose(A, B, rtol=tol, atol=tol * np.abs(B).max() * 1e-3)


def _col_scale(rows, j):
    vals = []
    for r in rows:
        try:
            vals.append(abs(float(r[j])))
        except (ValueError, IndexError):
            pass
    return max(vals) if vals else 0.0


def _out_of(manifest_path):
    for line in open(manifest_path).read().splitlines():
        if line.startswith("out="):
            return line[4:]
    return ""


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_cli_outputs_match_the_reference_cli(tmp_path, case):
    argv, rc_ref, conv = _argv(case)
    out = tmp_path / case
    with contextlib.redirect_stderr(io.StringIO()):
        rc = cli.main(argv + ["--out", str(out)])
    assert rc == rc_ref
    _compare_dir(str(out), os.path.join(GOLD, case), conv)
    if argv[0] in ("eigs", "variance"):
        assert (out / "diagnostics.log").read_text().startswith("iterations=")


# --------------------------------------------- reference CLI behaviours beyond the fixtures
def _quiet_main(argv):
    with contextlib.redirect_stderr(io.StringIO()):
        return cli.main(argv)


@pytest.mark.gpu
def test_steady_eigs_leading_value(tmp_path):
    """test_cli.py:27-39: the first Ritz value of the steady problem is (bp/bn)/lambda_11^2."""
    import paper_1703_05638_b200 as lp
    out = tmp_path / "steady"
    assert _quiet_main(["eigs", "--problem", "steady-poisson", "--mode", "steady", "--n-side", "15",
                        "--m-a", "60", "--eps-eig", "1e-12", "--check-every", "100", "--k", "5",
                        "--out", str(out)]) == 0
    header, rows = _csv(out / "eigenvalues.csv")
    assert header == ["index", "ritz_value", "imag_part"]
    want = 1e-4 / lp.discrete_fd_eig(1, 1, lp.build_grid(15)) ** 2
    assert float(rows[0][1]) == pytest.approx(want, rel=1e-8)


@pytest.mark.gpu
def test_repeated_and_manifest_driven_runs_are_bitwise_identical(tmp_path):
    """test_cli.py:42-64: the same flags twice, and a rerun from the written manifest,
    reproduce eigenvalues.csv / ranks.csv / hessenberg.csv byte for byte."""
    flags = ["eigs", "--problem", "heat", "--n-side", "7", "--nt", "4", "--m-a", "15", "--eps-eig",
             "1e-10", "--check-every", "100", "--seed", "3", "--start", "random"]
    a, b, c = tmp_path / "a", tmp_path / "b", tmp_path / "c"
    assert _quiet_main(flags + ["--out", str(a)]) == 0
    assert _quiet_main(flags + ["--out", str(b)]) == 0
    assert _quiet_main(["eigs", "--config", str(a / "manifest.cfg"), "--out", str(c)]) == 0
    for name in ("eigenvalues.csv", "ranks.csv", "hessenberg.csv"):
        assert (a / name).read_bytes() == (b / name).read_bytes() == (c / name).read_bytes()


@pytest.mark.gpu
def test_variance_with_nothing_retained_is_the_prior(tmp_path):
    """test_cli.py:67-80: a vanishing noise weight leaves every eigenvalue below the retention
    threshold; the field is gamma everywhere and retained.csv has no rows."""
    out = tmp_path / "flat"
    assert _quiet_main(["variance", "--problem", "heat", "--n-side", "7", "--nt", "4", "--sensors",
                        "none", "--beta-ratio", "1e-12", "--m-a", "10", "--eps-eig", "1e-1",
                        "--check-every", "100", "--gamma-prior", "10", "--out", str(out)]) == 0
    _, rows = _csv(out / "variance.csv")
    np.testing.assert_allclose(np.array(rows, dtype=float), 10.0, rtol=1e-12)
    assert _csv(out / "retained.csv")[1] == []


@pytest.mark.gpu
def test_variance_minimum_lies_on_a_sensor(tmp_path):
    """test_cli.py:83-95 (heat 31^2, n_t 10, 3x3 sensors) and the PGM header."""
    import paper_1703_05638_b200 as lp
    out = tmp_path / "var31"
    assert _quiet_main(["variance", "--problem", "heat", "--n-side", "31", "--nt", "10", "--m-a", "25",
                        "--eps-eig", "1e-1", "--out", str(out)]) == 0
    _, rows = _csv(out / "variance.csv")
    field = np.array(rows, dtype=float).ravel()
    assert lp.make_sensor_layout_3x3(lp.build_grid(31)).mask[int(np.argmin(field))]
    assert (out / "variance.pgm").read_text().startswith("P2\n31 31\n255\n")


@pytest.mark.gpu
@pytest.mark.parametrize("argv", [
    ["oracle", "--problem", "convdiff", "--nu", "1e-2", "--n-side", "5", "--nt", "4", "--m-a", "100",
     "--eps-eig", "1e-12", "--check-every", "100"],
    ["oracle", "--problem", "heat", "--n-side", "4", "--nt", "3", "--sensors", "none", "--mode",
     "source", "--m-a", "60", "--eps-eig", "1e-14", "--check-every", "100"],
], ids=["convdiff", "source"])
def test_oracle_passes_for_convdiff_and_source_mode(tmp_path, argv):
    """test_cli.py:108-115, 219-225."""
    out = tmp_path / "orc"
    assert _quiet_main(argv + ["--out", str(out)]) == 0
    assert "result=PASS" in (out / "oracle_report.txt").read_text()


def test_oracle_refuses_instances_above_the_dense_cap(tmp_path):
    """test_cli.py:126-129: exit code 2 (configuration error), decided on the host."""
    assert _quiet_main(["oracle", "--problem", "heat", "--n-side", "63", "--nt", "30",
                        "--out", str(tmp_path / "big")]) == 2


def test_sweep_rejects_an_unknown_axis(tmp_path):
    """test_cli.py:157-160."""
    assert _quiet_main(["sweep", "--axis", "bogus", "--values", "1,2", "--out", str(tmp_path / "x")]) == 2


@pytest.mark.gpu
def test_sweep_orders_points_and_survives_a_bad_one(tmp_path):
    """test_cli.py:132-154: summary.csv header and point labels, the leading eigenvalue grows as
    nu shrinks, one directory per point; an invalid point is recorded as ERROR, the sweep goes on
    and the exit code is 3."""
    out = tmp_path / "sweep"
    assert _quiet_main(["sweep", "--axis", "nu", "--values", "1e-1,1e-2,1e-3", "--problem", "convdiff",
                        "--n-side", "15", "--nt", "6", "--m-a", "25", "--eps-eig", "1e-1",
                        "--out", str(out)]) == 0
    header, rows = _csv(out / "summary.csv")
    assert header == ["point", "iterations_to_threshold", "max_rank", "largest_eig"]
    assert [r[0] for r in rows] == ["1e-1", "1e-2", "1e-3"]
    top = [float(r[3]) for r in rows]
    assert top[0] < top[1] < top[2]
    for r in rows:
        assert (out / f"nu_{r[0]}" / "eigenvalues.csv").exists()
    bad = tmp_path / "sweepfail"
    assert _quiet_main(["sweep", "--axis", "nu", "--values", "1e-2,-1.0", "--problem", "convdiff",
                        "--n-side", "7", "--nt", "4", "--m-a", "10", "--out", str(bad)]) == 3
    _, rows = _csv(bad / "summary.csv")
    assert rows[0][0] == "1e-2" and rows[1][1] == "ERROR"


@pytest.mark.gpu
def test_manifest_lists_every_reference_key_and_notes_degraded_sensors(tmp_path):
    """test_cli.py:193-208: one key=value line per configuration field; a 3x3 layout on a grid
    too coarse for it is replaced and the manifest says so."""
    out = tmp_path / "mani"
    assert _quiet_main(["eigs", "--problem", "heat", "--n-side", "7", "--nt", "3", "--sensors",
                        "grid3x3", "--m-a", "5", "--check-every", "100", "--out", str(out)]) == 0
    text = (out / "manifest.cfg").read_text()
    for s in cli.SETTINGS:
        if not s.extension:
            assert f"{s.key}=" in text, s.key
    assert "under-resolved" in text


@pytest.mark.gpu
def test_source_mode_eigs_writes_ranks_and_singular_values(tmp_path):
    """test_cli.py:228-239."""
    out = tmp_path / "src"
    assert _quiet_main(["eigs", "--problem", "heat", "--n-side", "9", "--nt", "6", "--sensors", "none",
                        "--mode", "source", "--m-a", "10", "--check-every", "100", "--out", str(out)]) == 0
    _, rows = _csv(out / "ranks.csv")
    assert len(rows) == 10 and all(int(r[1]) >= 1 for r in rows)
    header, sig = _csv(out / "singular_values.csv")
    assert header == ["vector", "index", "sigma"]
    first = [float(r[2]) for r in sig if r[0] == "0"]
    assert first and all(a >= b for a, b in zip(first, first[1:]))

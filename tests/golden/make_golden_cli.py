"""Fixtures for the CLI parity tests: runs the REFERENCE's own command line
(imported read-only from /root/reference in the build container) on small
configurations and stores its output files under tests/golden/cli/<case>/.
Timings (diagnostics.log) are not kept.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cli.py
"""
import contextlib
import io
import os
import shutil
import sys
import tempfile

sys.path.insert(0, "/root/reference/pkg/src")
from lrpostcov import cli  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = {
    "eigs_heat_ic": ["eigs", "--n-side", "13", "--nt", "10", "--m-a", "40", "--k", "12", "--seed", "3",
                     "--start", "random"],
    "eigs_heat_full": ["eigs", "--n-side", "10", "--nt", "6", "--m-a", "24", "--sensors", "none", "--start", "random"],
    "variance_custom": ["variance", "--n-side", "15", "--nt", "8", "--m-a", "30", "--gamma-prior", "2.5",
                        "--sensors", "custom:0.3,0.3,0.2;0.7,0.6,0.15", "--eps-eig", "1e-3"],
    "eigs_source": ["eigs", "--mode", "source", "--n-side", "9", "--nt", "6", "--m-a", "20", "--k", "6",
                    "--start", "random", "--seed", "1", "--r-max", "12"],
    "eigs_convdiff": ["eigs", "--problem", "convdiff", "--nu", "0.05", "--wind", "0.6,-0.8",
                      "--n-side", "12", "--nt", "8", "--m-a", "30", "--k", "8"],
    "eigs_steady": ["eigs", "--problem", "steady-poisson", "--mode", "steady", "--n-side", "9",
                    "--m-a", "30", "--k", "6", "--start", "random"],
    "oracle_heat": ["oracle", "--n-side", "7", "--nt", "5", "--m-a", "100", "--eps-eig", "1e-12",
                    "--check-every", "100"],
    "oracle_bad_truncation": ["oracle", "--n-side", "7", "--nt", "5", "--eps0", "0.5", "--m-a", "100",
                              "--eps-eig", "1e-12", "--check-every", "100"],
    "sweep_nu": ["sweep", "--problem", "convdiff", "--n-side", "9", "--nt", "5", "--m-a", "30",
                 "--axis", "nu", "--values", "0.01,0.1"],
}

for name, argv in CASES.items():
    dst = os.path.join(HERE, "cli", name)
    shutil.rmtree(dst, ignore_errors=True)
    with tempfile.TemporaryDirectory() as tmp:
        rc = cli.main(argv + ["--out", tmp])
        for root, _, files in os.walk(tmp):
            for f in files:
                if f == "diagnostics.log":
                    continue
                rel = os.path.relpath(os.path.join(root, f), tmp)
                os.makedirs(os.path.dirname(os.path.join(dst, rel)), exist_ok=True)
                text = open(os.path.join(root, f)).read().replace(tmp, "OUT")
                open(os.path.join(dst, rel), "w").write(text)
    # how many leading Ritz values are converged: stable (1e-9 of the largest) when the
    # same run gets 6 more Arnoldi steps — only those are comparable across implementations
    # (unconverged Ritz values and late Hessenberg columns are rounding-sensitive)
    conv = -1
    if argv[0] in ("eigs", "variance"):
        def ritz(extra):
            a = list(argv)
            i = a.index("--m-a")
            a[i + 1] = str(int(a[i + 1]) + extra)
            with tempfile.TemporaryDirectory() as t2:
                cli.main(a + ["--out", t2, "--k", "1000"])
                rows = open(os.path.join(t2, "eigenvalues.csv")).read().splitlines()[1:]
            return [float(r.split(",")[1]) for r in rows]
        a0, a1 = ritz(0), ritz(6)
        conv = 0
        for x, y in zip(a0, a1):
            if abs(x - y) > 1e-9 * abs(a0[0]):
                break
            conv += 1
    open(os.path.join(dst, "argv.txt"), "w").write(" ".join(argv) + f"\nrc={rc}\nconverged={conv}\n")
    print(name, "rc", rc, "converged", conv)
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    cli.main(["analytic", "--n-side", "6", "--k", "8"])
os.makedirs(os.path.join(HERE, "cli", "analytic"), exist_ok=True)
open(os.path.join(HERE, "cli", "analytic", "stdout.txt"), "w").write(buf.getvalue())

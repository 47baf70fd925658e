"""Command line over the device backend: the reference's experiment driver
(lrpostcov/cli.py:43-604) — same subcommands (eigs, variance, oracle, sweep,
analytic), the same flat key=value configuration with the precedence
flag > environment (LRPOSTCOV_*) > config file > default, the same exit codes
(0 ok / PASS, 2 configuration error, 3 numerical failure, 4 oracle FAIL) and
the same output files with 17 significant digits (manifest.cfg,
eigenvalues.csv, ranks.csv, hessenberg.csv, singular_values.csv,
diagnostics.log, variance.csv, variance.pgm, retained.csv,
oracle_report.txt, summary.csv), so a manifest written by either
implementation drives the other.

Everything is derived from ONE table of settings (`SETTINGS`): defaults, value
parsers, manifest formatting, environment names and the argparse flags.  The
keys after `out` are extensions for the BASELINE configurations;
left at their defaults they are not written to the manifest, which then stays
byte-identical to the reference's.

    python -m paper_1703_05638_b200.cli eigs --n-side 31 --nt 30 --out run1
"""

from __future__ import annotations

import argparse
import os
import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import dense, discretize, hessian, posterior
from .arnoldi import StopRule, lr_arnoldi, start_vector
from .errors import InvalidConfigError, NumericalError
from .forward import SpaceTimeOperator
from .lowrank import TruncationPolicy, lr_from_dense, lr_singular_values, lr_to_dense
from .posterior import write_variance_csv, write_variance_pgm  # noqa: F401 (used by cmd_variance)

ENV_PREFIX = "LRPOSTCOV_"
PROBLEMS = ("heat", "convdiff", "steady-poisson")
MODES = (hessian.MODE_IC, hessian.MODE_SOURCE, hessian.MODE_STEADY)


# ------------------------------------------------------------------ settings
def _as_int(key, raw):
    try:
        return int(raw)
    except ValueError as exc:
        raise InvalidConfigError(f"bad value for {key}: {raw!r}") from exc


def _as_float(key, raw):
    try:
        return float(raw)
    except ValueError as exc:
        raise InvalidConfigError(f"bad value for {key}: {raw!r}") from exc


def _as_text(key, raw):
    return raw


def _as_wind(key, raw):
    parts = raw.split(",")
    if len(parts) not in (2, 3):
        raise InvalidConfigError(f"wind needs two components, got {raw!r}")
    return tuple(_as_float(key, p) for p in parts)


def _as_cap(key, raw):
    return None if raw.lower() in ("none", "") else _as_int(key, raw)


def _show(value) -> str:
    if value is None:
        return "none"
    if isinstance(value, tuple):
        return ",".join(f"{v:.17g}" for v in value)
    if isinstance(value, float):
        return f"{value:.17g}"
    return str(value)


@dataclass(frozen=True)
class Setting:
    key: str
    default: object
    parse: object
    extension: bool = False    # beyond the reference's RunConfig (cli.py:43-67)
    choices: tuple | None = None

    @property
    def flag(self) -> str:
        return "--" + self.key.replace("_", "-")


SETTINGS = (
    Setting("problem", "heat", _as_text, choices=PROBLEMS),
    Setting("n_side", 31, _as_int),
    Setting("nt", 30, _as_int),
    Setting("final_time", 1.0, _as_float),
    Setting("nu", 1e-2, _as_float),
    Setting("wind", (0.0, 1.0), _as_wind),
    Setting("beta_ratio", 1e4, _as_float),
    Setting("gamma_mode", "scalar", _as_text, choices=("scalar", "beta")),
    Setting("gamma_prior", 10.0, _as_float),
    Setting("beta_prior", 1.0, _as_float),
    Setting("sensors", "grid3x3", _as_text),
    Setting("eps0", 1e-8, _as_float),
    Setting("r_max", None, _as_cap),
    Setting("eps_eig", 1e-1, _as_float),
    Setting("m_a", 100, _as_int),
    Setting("check_every", 10, _as_int),
    Setting("mode", "ic", _as_text, choices=MODES),
    Setting("start", "ones", _as_text, choices=("ones", "random")),
    Setting("on_breakdown", "stop", _as_text, choices=("stop", "restart")),
    Setting("seed", 0, _as_int),
    Setting("compress_every", 4, _as_int),
    Setting("k", 50, _as_int),
    Setting("out", "out", _as_text),
    # ---- extensions for the BASELINE configurations
    Setting("dim", 2, _as_int, extension=True),                  # 3: 7-point FD on the cube
    Setting("stencil", "fd", _as_text, extension=True, choices=("fd", "q1")),
    Setting("wind_field", "const", _as_text, extension=True, choices=("const", "rotating")),
    Setting("scheme", "upwind", _as_text, extension=True, choices=("upwind", "galerkin")),
    Setting("noise_sigma", 0.0, _as_float, extension=True),      # > 0: pointwise weight 1/sigma^2 (D1)
    Setting("prior_delta", 0.0, _as_float, extension=True),      # operator prior (delta I + gamma L)^-2
    Setting("prior_gamma", 0.0, _as_float, extension=True),
    Setting("obs_every", 1, _as_int, extension=True),            # sensors read every k-th step (D8)
)
_BY_KEY = {s.key: s for s in SETTINGS}


class RunConfig:
    """Resolved configuration: one attribute per SETTINGS entry (immutable by convention)."""

    __slots__ = tuple(s.key for s in SETTINGS)

    def __init__(self, **values):
        for s in SETTINGS:
            object.__setattr__(self, s.key, values.pop(s.key, s.default))
        if values:
            raise InvalidConfigError(f"unknown configuration key {next(iter(values))!r}")

    def __setattr__(self, key, value):
        raise AttributeError("RunConfig is read-only; use .replace()")

    def replace(self, **updates) -> "RunConfig":
        vals = {s.key: getattr(self, s.key) for s in SETTINGS}
        for k in updates:
            if k not in _BY_KEY:
                raise InvalidConfigError(f"unknown configuration key {k!r}")
        vals.update(updates)
        return RunConfig(**vals)

    def items(self):
        return [(s.key, getattr(self, s.key)) for s in SETTINGS]


def parse_value(key: str, raw: str):
    if key not in _BY_KEY:
        raise InvalidConfigError(f"unknown configuration key {key!r}")
    return _BY_KEY[key].parse(key, raw.strip())


def load_config_file(path) -> dict:
    try:
        text = Path(path).read_text()
    except OSError as exc:
        raise InvalidConfigError(f"cannot read config file {path}: {exc}") from exc
    found = {}
    for no, line in enumerate(text.splitlines(), start=1):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, sep, raw = line.partition("=")
        if not sep:
            raise InvalidConfigError(f"{path}:{no}: expected key=value, got {line!r}")
        found[key.strip()] = parse_value(key.strip(), raw)
    return found


def env_overrides(environ=None) -> dict:
    environ = os.environ if environ is None else environ
    return {s.key: parse_value(s.key, environ[ENV_PREFIX + s.key.upper()])
            for s in SETTINGS if ENV_PREFIX + s.key.upper() in environ}


def validate_config(cfg: RunConfig) -> None:
    for s in SETTINGS:
        if s.choices and getattr(cfg, s.key) not in s.choices:
            raise InvalidConfigError(f"{s.key} must be one of {s.choices}, got {getattr(cfg, s.key)!r}")
    steady = cfg.problem == "steady-poisson"
    if steady != (cfg.mode == hessian.MODE_STEADY):
        raise InvalidConfigError("problem steady-poisson and mode=steady go together")
    if cfg.n_side < 2:
        raise InvalidConfigError(f"n_side must be >= 2, got {cfg.n_side}")
    if cfg.nt < 1:
        raise InvalidConfigError(f"nt must be >= 1, got {cfg.nt}")
    if not 0 < cfg.eps0 < 1:
        raise InvalidConfigError(f"eps0 must lie in (0, 1), got {cfg.eps0}")
    if min(cfg.eps_eig, cfg.beta_ratio) <= 0 or min(cfg.m_a, cfg.check_every) < 1:
        raise InvalidConfigError("eps_eig, beta_ratio, m_a, check_every must be positive")
    sens = cfg.sensors
    if not (sens in ("none", "grid3x3") or sens.startswith(("custom:", "subgrid:"))):
        raise InvalidConfigError(f"unknown sensors setting {sens!r}")
    if cfg.dim not in (2, 3) or cfg.obs_every < 1 or cfg.noise_sigma < 0 or cfg.prior_gamma < 0:
        raise InvalidConfigError("dim must be 2 or 3; obs_every >= 1; noise_sigma, prior_gamma >= 0")


def resolve_config(file_path=None, env=None, flag_updates=None) -> RunConfig:
    """flag > environment > file > default, then validation (cli.py:130-142)."""
    layers = [load_config_file(file_path) if file_path is not None else {}, env_overrides(env)]
    flags = {k: (parse_value(k, v) if isinstance(v, str) else v)
             for k, v in (flag_updates or {}).items()}
    cfg = RunConfig()
    for layer in layers + [flags]:
        cfg = cfg.replace(**layer)
    validate_config(cfg)
    return cfg


def write_manifest(cfg: RunConfig, outdir: Path, notes: dict | None = None) -> None:
    lines = [f"{k}={_show(v)}" for k, v in cfg.items()
             if not (_BY_KEY[k].extension and v == _BY_KEY[k].default)]
    lines += [f"# {k}: {v}" for k, v in (notes or {}).items()]
    (outdir / "manifest.cfg").write_text("\n".join(lines) + "\n")


# ------------------------------------------------------------------- problem
@dataclass
class Problem:
    """A resolved configuration assembled on the device."""

    config: RunConfig
    grid: object
    spatial: object
    time: object
    K: object
    layout: object
    cov: object
    pol: TruncationPolicy
    ctx: hessian.HessianContext
    notes: dict


def _sensor_layout(cfg: RunConfig, grid, notes: dict):
    s = cfg.sensors
    if s == "none":
        lay = hessian.full_observation(grid)
    elif s == "grid3x3":
        try:
            lay = hessian.make_sensor_layout_3x3(grid)
        except InvalidConfigError:
            notes["sensors_resolved"] = "full (grid3x3 under-resolved)"
            lay = hessian.full_observation(grid)
    elif s.startswith("subgrid:"):
        return hessian.make_sensor_subgrid(grid, _as_int("sensors", s.split(":", 1)[1]),
                                           time_every=cfg.obs_every)
    else:
        patches = []
        for item in s.split(":", 1)[1].split(";"):
            nums = item.split(",")
            if len(nums) != 3:
                raise InvalidConfigError(f"custom sensor patch needs cx,cy,side, got {item!r}")
            patches.append(tuple(float(x) for x in nums))
        lay = hessian.make_sensor_layout(patches, grid)
    if cfg.obs_every > 1:
        lay = hessian.SensorLayout(lay.patches, lay.mask, time_every=cfg.obs_every)
    return lay


def build_problem(cfg: RunConfig) -> Problem:
    notes: dict = {}
    grid = discretize.build_grid(cfg.n_side, cfg.dim)
    maker = hessian.CovarianceSpec.from_gamma if cfg.gamma_mode == "scalar" \
        else hessian.CovarianceSpec.from_beta
    cov = maker(cfg.gamma_prior if cfg.gamma_mode == "scalar" else cfg.beta_prior,
                cfg.beta_ratio, grid)
    pol = TruncationPolicy(eps0=cfg.eps0, r_max=cfg.r_max)
    if cfg.problem == "steady-poisson":
        spatial = discretize.assemble_heat(grid)
        ctx = hessian.HessianContext(mode=hessian.MODE_STEADY, operator=None, layout=None, cov=cov,
                                     pol=pol, spatial=spatial)
        return Problem(cfg, grid, spatial, None, None, None, cov, pol, ctx, notes)
    if cfg.problem == "heat":
        spatial = discretize.assemble_heat(grid, cfg.stencil)
    else:
        spatial = discretize.assemble_convdiff(grid, cfg.nu, cfg.wind, field=cfg.wind_field,
                                               scheme=cfg.scheme)
    time = discretize.build_time_grid(cfg.nt, cfg.final_time)
    K = SpaceTimeOperator(spatial, time)
    if cfg.noise_sigma > 0 or cfg.prior_gamma > 0:
        bn = cov.beta_noise if cfg.noise_sigma <= 0 \
            else 1.0 / (cfg.noise_sigma ** 2 * time.tau * grid.m_scale)
        cov = hessian.CovarianceSpec(bn, cov.beta_prior, cov.gamma_prior,
                                     prior_delta=cfg.prior_delta if cfg.prior_gamma > 0 else 0.0,
                                     prior_gamma=cfg.prior_gamma)
    layout = _sensor_layout(cfg, grid, notes)
    ctx = hessian.HessianContext(mode=cfg.mode, operator=K, layout=layout, cov=cov, pol=pol,
                                 compress_every=cfg.compress_every)
    return Problem(cfg, grid, spatial, time, K, layout, cov, pol, ctx, notes)


def _start(cfg: RunConfig, problem: Problem):
    return start_vector(problem.grid.n_x, problem.time.n_t if problem.time else None,
                        mode=cfg.mode, start=cfg.start, seed=cfg.seed)


# ---------------------------------------------------------------------- runs
@dataclass
class EigsRun:
    config: RunConfig
    problem: Problem
    result: object


def run_eigs(cfg: RunConfig, force_restart: bool = False) -> EigsRun:
    problem = build_problem(cfg)
    mode_break = "restart" if force_restart else cfg.on_breakdown
    m_a = cfg.m_a
    if cfg.mode != hessian.MODE_SOURCE:
        # a dense Krylov space cannot exceed n_x; restarts use up slots (cli.py:276-281)
        m_a = min(m_a, problem.ctx.n_param + (8 if mode_break == "restart" else 0))
    stop = StopRule(m_a=m_a, eps_eig=cfg.eps_eig, check_every=cfg.check_every,
                    on_breakdown=mode_break, restart_seed=cfg.seed)
    res = lr_arnoldi(problem.ctx.apply, _start(cfg, problem), problem.pol, stop,
                     rank_source=problem.ctx.rank_trace)
    return EigsRun(cfg, problem, res)


def run_variance(cfg: RunConfig, retain: float | None = None):
    if cfg.mode == hessian.MODE_SOURCE:
        raise InvalidConfigError(
            "the variance field is defined for spatial parameter modes (ic, steady)")
    run = run_eigs(cfg)
    summary = posterior.build_summary(
        run.result.ritz_values, run.result.ritz_vectors, gamma_prior=run.problem.cov.gamma_prior,
        eps_eig=cfg.eps_eig if retain is None else retain, n_x=run.problem.grid.n_x,
        prior=getattr(run.problem.ctx, "prior", None))
    return run, summary


# ------------------------------------------------------------------- writers
def _table(path: Path, header: str, rows) -> None:
    path.write_text("".join(line + "\n" for line in [header, *rows]))


def write_eigs_outputs(run: EigsRun, outdir: Path) -> None:
    res, cfg = run.result, run.config
    vals = res.ritz_values
    k = min(cfg.k, len(vals))
    _table(outdir / "eigenvalues.csv", "index,ritz_value,imag_part",
           [f"{i},{vals[i].real:.17g},{vals[i].imag:.17g}" for i in range(k)])
    _table(outdir / "ranks.csv", "iteration,max_intermediate_rank",
           [f"{j},{r}" for j, r in enumerate(res.rank_trace, start=1)])
    H = res.H
    m = H.shape[1]
    _table(outdir / "hessenberg.csv", "i,j,value",
           [f"{i},{j},{H[i, j]:.17g}" for j in range(m) for i in range(min(j + 2, m + 1))])
    if cfg.mode == hessian.MODE_SOURCE:
        _table(outdir / "singular_values.csv", "vector,index,sigma",
               [f"{v},{i},{s:.17g}" for v in range(k)
                for i, s in enumerate(lr_singular_values(res.ritz_vectors[v]))])
    log = [f"iterations={res.iterations} breakdown={res.breakdown} "
           f"converged_count={res.converged_count}"]
    log += [f"iter={j} h_subdiag={h:.6e} max_rank={r} seconds={t:.4f}"
            for j, h, r, t in res.diagnostics]
    (outdir / "diagnostics.log").write_text("\n".join(log) + "\n")


def _outdir(cfg: RunConfig) -> Path:
    d = Path(cfg.out)
    d.mkdir(parents=True, exist_ok=True)
    return d


# ------------------------------------------------------------------ commands
def cmd_eigs(cfg: RunConfig) -> int:
    d = _outdir(cfg)
    run = run_eigs(cfg)
    write_eigs_outputs(run, d)
    write_manifest(cfg, d, run.problem.notes)
    return 0


def cmd_variance(cfg: RunConfig) -> int:
    if cfg.dim != 2:
        raise InvalidConfigError("the variance grid writers are 2-D")
    d = _outdir(cfg)
    run, summary = run_variance(cfg)
    write_eigs_outputs(run, d)
    write_variance_csv(summary.variance_field, cfg.n_side, d / "variance.csv")
    write_variance_pgm(summary.variance_field, cfg.n_side, summary.gamma_prior, d / "variance.pgm")
    _table(d / "retained.csv", "lambda,lambda_tilde",
           [f"{a:.17g},{b:.17g}" for a, b in zip(summary.eigenvalues, summary.filters)])
    write_manifest(cfg, d, run.problem.notes)
    return 0


def _dense_hessian(problem: Problem):
    cfg, cov = problem.config, problem.cov
    L = problem.spatial.L.toarray()
    if cfg.mode == hessian.MODE_STEADY:
        return dense.dense_misfit_steady(L, cov.beta_noise, cov.beta_prior)
    build = dense.dense_misfit_ic if cfg.mode == hessian.MODE_IC else dense.dense_misfit_source
    return build(L, problem.grid.m_scale, problem.time.tau, problem.time.n_t, problem.layout.mask,
                 cov.beta_noise, cov.gamma_prior)


def _stacked_apply(problem: Problem):
    """The matrix-free apply on stacked dense vectors (source mode: vec of the field)."""
    if problem.config.mode != hessian.MODE_SOURCE:
        return problem.ctx.apply
    shape = (problem.grid.n_x, problem.time.n_t)

    def apply(v):
        field_in = lr_from_dense(np.asarray(v, dtype=float).reshape(shape, order="F"), problem.pol)
        return lr_to_dense(problem.ctx.apply(field_in)).reshape(-1, order="F")

    return apply


def run_oracle(cfg: RunConfig, retain: float = 1e-8, top_k: int = 10):
    """Low-rank path against the dense GPU brute force (cli.py:415-470)."""
    if cfg.prior_gamma > 0 or cfg.obs_every > 1 or cfg.dim != 2:
        raise InvalidConfigError("the dense oracle covers the reference's scalar-prior 2-D instances")
    source = cfg.mode == hessian.MODE_SOURCE
    dim = cfg.n_side ** cfg.dim * (cfg.nt if source else 1)
    if dim > dense.DENSE_DIM_CAP:   # a configuration error, decided before any device work
        raise InvalidConfigError(
            f"dense oracle dimension {dim} exceeds the cap {dense.DENSE_DIM_CAP}")
    probe = build_problem(cfg)
    Hd, asym = _dense_hessian(probe)
    hv = dense.hv_agreement(_stacked_apply(probe), Hd, n_probe=20, seed=cfg.seed)
    run = run_eigs(cfg.replace(m_a=min(cfg.m_a, dim + 8)), force_restart=True)
    res = run.result
    k = min(top_k, dim, len(res.ritz_values))
    d_vals, d_vecs = dense.dense_eig_top(Hd, k)
    cols = [lr_to_dense(v).reshape(-1, order="F") if source else np.asarray(v)
            for v in res.ritz_vectors[:k]]
    lr_var = dn_var = None
    if not source:
        summ = posterior.build_summary(res.ritz_values, res.ritz_vectors,
                                       gamma_prior=probe.cov.gamma_prior, eps_eig=retain, n_x=dim)
        lr_var, dn_var = summ.variance_field, dense.dense_posterior_diag(Hd, probe.cov.gamma_prior)
    report = dense.compare(res.ritz_values.real, np.column_stack(cols), d_vals, d_vecs, Hd=Hd,
                           lr_variance=lr_var, dense_variance=dn_var, hv_rel_error=hv)
    report.tolerances["asymmetry"] = asym
    return run.problem, res, report


def cmd_oracle(cfg: RunConfig) -> int:
    d = _outdir(cfg)
    problem, _, report = run_oracle(cfg)
    (d / "oracle_report.txt").write_text(report.as_text())
    write_manifest(cfg, d, problem.notes)
    return 0 if report.passed else 4


SWEEP_AXES = {"nt": "nt", "n-side": "n_side", "nu": "nu", "beta-ratio": "beta_ratio",
              "eps0": "eps0", "eps-eig": "eps_eig"}


def cmd_sweep(cfg: RunConfig, axis: str, values: list) -> int:
    if axis not in SWEEP_AXES:
        raise InvalidConfigError(f"sweep axis must be one of {sorted(SWEEP_AXES)}, got {axis!r}")
    if not values:
        raise InvalidConfigError("sweep needs a nonempty list of axis values")
    top = _outdir(cfg)
    rows, any_failed = [], False
    for raw in values:
        try:  # every point is an independent run in its own directory
            point = cfg.replace(**{SWEEP_AXES[axis]: parse_value(SWEEP_AXES[axis], raw),
                                   "out": str(top / f"{axis}_{raw}")})
            validate_config(point)
            pd = _outdir(point)
            run = run_eigs(point)
            write_eigs_outputs(run, pd)
            write_manifest(point, pd, run.problem.notes)
            r = run.result
            lead = r.ritz_values[0].real if len(r.ritz_values) else 0.0
            rows.append(f"{raw},{r.iterations},{max(r.rank_trace, default=0)},{lead:.17g}")
        except (InvalidConfigError, NumericalError) as exc:
            any_failed = True
            rows.append(f"{raw},ERROR,ERROR,ERROR")
            print(f"sweep point {axis}={raw} failed: {exc}", file=sys.stderr)
    _table(top / "summary.csv", "point,iterations_to_threshold,max_rank,largest_eig", rows)
    write_manifest(cfg, top, {"sweep_axis": axis, "sweep_values": ",".join(values)})
    return 3 if any_failed else 0


def cmd_analytic(cfg: RunConfig) -> int:
    grid = discretize.build_grid(cfg.n_side)
    pairs = sorted(((m, n) for m in range(1, grid.n_side + 1) for n in range(1, grid.n_side + 1)),
                   key=lambda mn: discretize.discrete_fd_eig(mn[0], mn[1], grid))
    print("m,n,lambda_analytic,lambda_discrete,mu_steady")
    for m, n in pairs[: min(cfg.k, len(pairs))]:
        lam = discretize.discrete_fd_eig(m, n, grid)
        print(f"{m},{n},{discretize.analytic_poisson_eig(m, n):.17g},{lam:.17g},"
              f"{(1.0 / cfg.beta_ratio) / lam ** 2:.17g}")
    return 0


# ---------------------------------------------------------------- entry point
_COMMANDS = {
    "eigs": ("compute the dominant misfit-Hessian eigenvalues", cmd_eigs),
    "variance": ("compute the pointwise posterior variance field", cmd_variance),
    "oracle": ("compare the low-rank path against a dense reference", cmd_oracle),
    "sweep": ("run a parameter sweep", None),
    "analytic": ("print analytic/discrete Laplacian eigenvalue tables", cmd_analytic),
}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="lrpostcov",
        description="Low-rank posterior covariance approximation for space-time Bayesian "
                    "inverse problems (B200 device backend)")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (text, _) in _COMMANDS.items():
        p = sub.add_parser(name, help=text)
        p.add_argument("--config", help="key=value config file (e.g. a manifest)")
        for s in SETTINGS:  # values stay raw strings here; resolve_config parses them
            p.add_argument(s.flag, dest=s.key, choices=s.choices if s.choices else None)
        if name == "sweep":
            p.add_argument("--axis", required=True, help=f"one of {sorted(SWEEP_AXES)}")
            p.add_argument("--values", required=True, help="comma-separated axis values")
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        flags = {s.key: getattr(args, s.key) for s in SETTINGS if getattr(args, s.key) is not None}
        cfg = resolve_config(file_path=args.config, flag_updates=flags)
        if args.command == "sweep":
            return cmd_sweep(cfg, args.axis, [v for v in args.values.split(",") if v])
        return _COMMANDS[args.command][1](cfg)
    except InvalidConfigError as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return 2
    except NumericalError as exc:
        print(f"numerical failure: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())

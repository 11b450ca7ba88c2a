"""Run configuration of the reference CLI (config.hpp:18-282): the
line-oriented ``key = value`` format with ``[section]`` headers and full-line
``#`` comments, the same schema, defaults, validation and error messages
(std::runtime_error -> ConfigError).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Tuple

from .api import IntegratorConfig


class ConfigError(RuntimeError):
    """config.hpp parse errors (std::runtime_error)."""


@dataclass
class RunConfig:
    """config.hpp:24-50. Zero / NaN sentinels mean "use the scenario's default"."""
    scenario: str = ""
    scenario_params: Dict[str, float] = field(default_factory=dict)
    nx: int = 0
    ny: int = 0
    t0: float = math.nan
    t_final: float = math.nan
    threads: int = 0
    integrator: IntegratorConfig = field(default_factory=IntegratorConfig)
    tolerances_set: bool = False
    output_dir: str = "out"
    gauges_set: bool = False
    gauges: List[Tuple[float, float]] = field(default_factory=list)
    snapshots_set: bool = False
    snapshot_times: List[float] = field(default_factory=list)
    conservation_stride: int = 1
    cross_section_set: bool = False
    cross_section_y: float = 0.0
    resolutions: List[int] = field(default_factory=list)
    converge_ny: int = 0
    bench_resolutions: List[int] = field(default_factory=lambda: [128, 181, 256, 362, 512])
    bench_repetitions: int = 50
    bench_warmups: int = 5


_SCHEMA = {
    "run": {"scenario", "nx", "ny", "t0", "t_final", "threads"},
    "scenario": set(),  # free-form numeric parameters
    "integrator": {"abs_tol", "rel_tol", "dt_initial", "dt_max", "fixed_dt", "max_steps", "safety", "growth_cap",
                   "shrink_floor"},
    "output": {"directory", "gauges", "snapshot_times", "conservation_stride", "cross_section_y"},
    "converge": {"resolutions", "ny"},
    "bench": {"resolutions", "repetitions", "warmups"},
}


def _trim(s: str) -> str:
    """config.hpp:54-60: strips spaces, tabs and carriage returns."""
    return s.strip(" \t\r")


def _strtod(t: str):
    """The whole-string std::strtod acceptance of parse_double: decimal and
    hex floats, inf/nan, optional sign; None when not fully consumed."""
    try:
        return float(t)
    except ValueError:
        pass
    if t.lstrip("+-")[:2].lower() == "0x":
        try:
            return float.fromhex(t)
        except ValueError:
            return None
    return None


def parse_double(where: str, text: str) -> float:
    t = _trim(text)
    v = _strtod(t) if t and "_" not in t else None
    if v is None:
        raise ConfigError(f"config: {where}: expected a number, got '{text}'")
    return v


def parse_int(where: str, text: str) -> int:
    v = parse_double(where, text)
    r = float(round(v)) if math.isfinite(v) else v
    if not (abs(v - r) <= 0.0):
        raise ConfigError(f"config: {where}: expected an integer, got '{text}'")
    return int(r)


def parse_double_list(where: str, text: str) -> List[float]:
    out = [parse_double(where, p) for p in (_trim(x) for x in text.split(",")) if p]
    if not out:
        raise ConfigError(f"config: {where}: expected a list of numbers")
    return out


def parse_int_list(where: str, text: str) -> List[int]:
    out = []
    for v in parse_double_list(where, text):
        r = float(round(v)) if math.isfinite(v) else v
        if not (abs(v - r) <= 0.0):
            raise ConfigError(f"config: {where}: expected integers")
        out.append(int(r))
    return out


def parse_pair_list(where: str, text: str) -> List[Tuple[float, float]]:
    """Gauge list: semicolon-separated pairs "x, y" (config.hpp:118-134)."""
    out = []
    for pair in text.split(";"):
        p = _trim(pair)
        if not p:
            continue
        xy = parse_double_list(where, p)
        if len(xy) != 2:
            raise ConfigError(f"config: {where}: each gauge needs exactly x, y")
        out.append((xy[0], xy[1]))
    if not out:
        raise ConfigError(f"config: {where}: expected 'x1, y1; x2, y2; ...'")
    return out


def parse_config_text(text: str) -> RunConfig:
    """config.hpp:139-247. Unknown sections or keys are errors; [scenario]
    keys are validated later by the scenario registry."""
    cfg = RunConfig()
    section = ""
    for lineno, line in enumerate(text.split("\n"), start=1):
        s = _trim(line)
        if not s or s[0] == "#":
            continue
        at = f"line {lineno}"
        if s[0] == "[":
            if s[-1] != "]":
                raise ConfigError(f"config: {at}: malformed section header")
            section = _trim(s[1:-1])
            if section not in _SCHEMA:
                raise ConfigError(f"config: {at}: unknown section [{section}]")
            continue
        eq = s.find("=")
        if eq < 0:
            raise ConfigError(f"config: {at}: expected key = value")
        key, value = _trim(s[:eq]), _trim(s[eq + 1:])
        if not section:
            raise ConfigError(f"config: {at}: key outside any [section]")
        if not key:
            raise ConfigError(f"config: {at}: empty key")
        if section != "scenario" and key not in _SCHEMA[section]:
            raise ConfigError(f"config: {at}: unknown key '{key}' in section [{section}]")
        where = f"[{section}] {key}"
        ic = cfg.integrator
        if section == "run":
            if key == "scenario":
                cfg.scenario = value
            elif key == "nx":
                cfg.nx = parse_int(where, value)
            elif key == "ny":
                cfg.ny = parse_int(where, value)
            elif key == "t0":
                cfg.t0 = parse_double(where, value)
            elif key == "t_final":
                cfg.t_final = parse_double(where, value)
            elif key == "threads":
                cfg.threads = parse_int(where, value)
        elif section == "scenario":
            cfg.scenario_params[key] = parse_double(where, value)
        elif section == "integrator":
            if key in ("abs_tol", "rel_tol"):
                setattr(ic, key, parse_double(where, value))
                cfg.tolerances_set = True
            elif key == "max_steps":
                ic.max_steps = parse_int(where, value)
            else:
                setattr(ic, key, parse_double(where, value))
        elif section == "output":
            if key == "directory":
                cfg.output_dir = value
            elif key == "gauges":
                cfg.gauges = parse_pair_list(where, value)
                cfg.gauges_set = True
            elif key == "snapshot_times":
                cfg.snapshot_times = parse_double_list(where, value)
                cfg.snapshots_set = True
            elif key == "conservation_stride":
                cfg.conservation_stride = parse_int(where, value)
                if cfg.conservation_stride < 1:
                    raise ConfigError(f"config: {where}: stride must be >= 1")
            elif key == "cross_section_y":
                cfg.cross_section_y = parse_double(where, value)
                cfg.cross_section_set = True
        elif section == "converge":
            if key == "resolutions":
                cfg.resolutions = parse_int_list(where, value)
            elif key == "ny":
                cfg.converge_ny = parse_int(where, value)
        elif section == "bench":
            if key == "resolutions":
                cfg.bench_resolutions = parse_int_list(where, value)
            elif key == "repetitions":
                cfg.bench_repetitions = parse_int(where, value)
            elif key == "warmups":
                cfg.bench_warmups = parse_int(where, value)
    return cfg


def parse_config_file(path: str) -> RunConfig:
    """config.hpp:249-256"""
    try:
        with open(path, "r", newline="") as fh:
            text = fh.read()
    except OSError:
        raise ConfigError(f"config: cannot open '{path}'") from None
    return parse_config_text(text)


def apply_thread_env(cfg: RunConfig) -> None:
    """config.hpp:260-272: the config key wins over THREADS (host threads of
    the reference; recorded in run_meta.json, the device path ignores it)."""
    if cfg.threads > 0:
        return
    env = os.environ.get("THREADS")
    if env is not None:
        try:
            cfg.threads = parse_int("THREADS", env)
        except ConfigError:
            raise ConfigError("THREADS environment variable is not an integer") from None


__all__ = ["ConfigError", "RunConfig", "parse_config_text", "parse_config_file", "apply_thread_env"]

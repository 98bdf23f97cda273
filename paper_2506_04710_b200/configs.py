"""The five BASELINE.json workloads (C1..C5) with every unspecified choice
fixed: seeds, correction rank, RHS kind, GMRES
settings. Inputs are synthetic and seeded (include/tbt_gen.h); the paper's
geometries are not available."""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Config:
    name: str
    nx: int
    ny: int
    m: int
    nrhs: int
    rank: int        # diag + rank-r nine-component perturbations
    seed: int
    rhs: str         # "normal" | "delta_steered" | "ports"
    restart: int
    tol: float = 1e-8
    max_iter: int = 2000
    scale: float = 0.1

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.m


CONFIGS = {
    "C1": Config("C1", 4, 4, 24, 1, 4, 0, "normal", 30),
    "C2": Config("C2", 32, 32, 64, 1, 8, 2, "delta_steered", 50),
    "C3": Config("C3", 18, 9, 128, 162, 8, 3, "ports", 50),
    "C4": Config("C4", 64, 64, 128, 1, 8, 4, "normal", 50),
    "C5": Config("C5", 128, 128, 192, 1, 8, 5, "normal", 50),
}


def rhs_for(cfg: Config):
    from . import gen
    if cfg.rhs == "normal":
        return gen.rhs_normal(cfg.n, cfg.nrhs, cfg.seed)
    if cfg.rhs == "delta_steered":
        return gen.rhs_delta_steered(cfg.nx, cfg.ny, cfg.m, cfg.seed, 30.0)
    if cfg.rhs == "ports":
        return gen.rhs_ports(cfg.nx, cfg.ny, cfg.m, cfg.seed)[0]
    raise ValueError(cfg.rhs)

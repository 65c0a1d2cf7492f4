"""Problem setup: the reference's Scenario / DynamicsModel / RewardConfig
(scenario.hpp:17-30, dynamics.hpp:22-34, reward.hpp:13-19) as one value type,
the reference's generators (scenario.cpp:110-255) and the BASELINE configs.

Layouts are the reference's column-major ones, stored C-contiguous with the
column index first: ``starts[k]`` is robot k's start state (dx), ``goals[k]``
its goal position (pdim), ``obs_centers[o]`` obstacle o's centre.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

DIFFDRIVE, HOLO2D, HOLO3D, HOLO2D_VEL, HOLO3D_VEL, UNICYCLE = range(6)
KIND_NAMES = {DIFFDRIVE: "diffdrive", HOLO2D: "holo2d", HOLO3D: "holo3d",
              HOLO2D_VEL: "holo2d_vel", HOLO3D_VEL: "holo3d_vel", UNICYCLE: "unicycle"}
DIMS = {DIFFDRIVE: (4, 2, 2), HOLO2D: (4, 2, 2), HOLO3D: (6, 3, 3),
        HOLO2D_VEL: (2, 2, 2), HOLO3D_VEL: (3, 3, 3), UNICYCLE: (3, 2, 2)}  # dx, du, pdim
MAX_REJECTIONS = 10000  # scenario.cpp:14


@dataclass
class Problem:
    kind: int
    starts: np.ndarray            # (R, dx)
    goals: np.ndarray             # (R, pdim)
    horizon: int = 100            # OptimizerConfig::horizon (optimizer.hpp:17)
    dt: float = 0.1
    lower: np.ndarray | None = None
    upper: np.ndarray | None = None
    obs_centers: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))
    obs_radii: np.ndarray = field(default_factory=lambda: np.zeros((0,)))
    w_t: float = 2.0              # RewardConfig defaults (reward.hpp:14-18)
    epsilon: float = 0.05
    robot_radius: float = 0.1
    goal_tolerance: float = 0.1
    obstacle_weight: float = 2.0
    effort_weight: float = 0.0    # extension: 0 = reference reward
    name: str = ""

    def __post_init__(self):
        dx, du, pd = DIMS[self.kind]
        self.starts = np.ascontiguousarray(self.starts, dtype=np.float64).reshape(-1, dx)
        self.goals = np.ascontiguousarray(self.goals, dtype=np.float64).reshape(-1, pd)
        self.obs_centers = np.ascontiguousarray(self.obs_centers, dtype=np.float64).reshape(-1, pd)
        self.obs_radii = np.ascontiguousarray(self.obs_radii, dtype=np.float64).reshape(-1)
        if self.lower is None:
            self.lower = np.full(du, -2.0)  # DynamicsModel::make default ±2 (dynamics.hpp:33)
        if self.upper is None:
            self.upper = -np.asarray(self.lower, dtype=np.float64)
        self.lower = np.asarray(self.lower, dtype=np.float64).reshape(du)
        self.upper = np.asarray(self.upper, dtype=np.float64).reshape(du)

    @property
    def dims(self):
        return DIMS[self.kind]

    @property
    def dx(self):
        return DIMS[self.kind][0]

    @property
    def du(self):
        return DIMS[self.kind][1]

    @property
    def pdim(self):
        return DIMS[self.kind][2]

    @property
    def robots(self):
        return self.starts.shape[0]

    @property
    def elems(self):
        """R*du*T: size of one joint control sequence."""
        return self.robots * self.du * self.horizon

    def with_horizon(self, horizon: int) -> "Problem":
        return replace(self, horizon=horizon)


# ------------------------------------------------------------------ RNG
# The reference's generator discipline: std::mt19937_64(mix_seed(seed, tag))
# with std::uniform_real_distribution<double> (scenario.cpp:207-208).
MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def mix_seed(a: int, b: int, c: int | None = None) -> int:
    """rng.hpp:17-23"""
    r = splitmix64(splitmix64(a & MASK64) ^ ((0x9E3779B97F4A7C15 + b) & MASK64))
    return r if c is None else mix_seed(r, c)


class MT19937_64:
    """std::mt19937_64 ([rand.eng.mers], output fixed by the standard)."""

    def __init__(self, seed: int):
        mt = [seed & MASK64]
        for i in range(1, 312):
            prev = mt[-1]
            mt.append((6364136223846793005 * (prev ^ (prev >> 62)) + i) & MASK64)
        self.mt, self.idx = mt, 312

    def __call__(self) -> int:
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                y = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                v = mt[(i + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                mt[i] = v
            self.idx = 0
        z = self.mt[self.idx]
        self.idx += 1
        z ^= (z >> 29) & 0x5555555555555555
        z ^= (z << 17) & 0x71D67FFFEDA60000
        z ^= (z << 37) & 0xFFF7EEE000000000
        z ^= z >> 43
        return z & MASK64

    def canonical(self) -> float:
        r = float(self()) / 18446744073709551616.0
        return r if r < 1.0 else math.nextafter(1.0, 0.0)

    def uniform(self, a: float, b: float) -> float:
        """std::uniform_real_distribution<double>(a, b) in libstdc++."""
        return self.canonical() * (b - a) + a


# ------------------------------------------------------------ generators
def _start_state(kind: int, pos: np.ndarray, goal: np.ndarray) -> np.ndarray:
    """make_start_state (scenario.cpp:27-38): zero velocity; heading robots face their goal."""
    dx = DIMS[kind][0]
    x = np.zeros(dx)
    x[: len(pos)] = pos
    if kind in (DIFFDRIVE, UNICYCLE):
        x[2] = math.atan2(goal[1] - pos[1], goal[0] - pos[0])
    return x


def antipodal_circle(robots: int, diameter: float, kind: int, robot_radius: float = 0.1, **kw) -> Problem:
    """scenario.cpp:110-148: starts equally spaced on a circle, goals opposite."""
    if robots < 1:
        raise ValueError("antipodal_circle: needs at least one robot")
    if not diameter > 0:
        raise ValueError("antipodal_circle: diameter must be > 0")
    if DIMS[kind][2] != 2:
        raise ValueError("antipodal_circle: use antipodal_sphere for 3D")
    if robots >= 2 and diameter * math.sin(math.pi / robots) <= 2.0 * robot_radius:
        raise ValueError("antipodal_circle: starts closer than 2*R_a")
    radius = diameter / 2.0
    starts, goals = [], []
    for k in range(robots):
        angle = 2.0 * math.pi * k / robots
        pos = np.array([radius * math.cos(angle), radius * math.sin(angle)])
        goal = -pos
        goals.append(goal)
        starts.append(_start_state(kind, pos, goal))
    return Problem(kind, np.array(starts), np.array(goals), robot_radius=robot_radius,
                   name=f"antipodal-circle-{KIND_NAMES[kind]}-n{robots}", **kw)


def antipodal_sphere(robots: int, diameter: float, robot_radius: float = 0.1, kind: int = HOLO3D, **kw) -> Problem:
    """scenario.cpp:150-197: pole-to-pole golden-angle spiral, goals antipodal."""
    golden = math.pi * (3.0 - math.sqrt(5.0))
    unit = []
    for k in range(robots):
        z = 1.0 if robots == 1 else 1.0 - 2.0 * k / (robots - 1.0)
        ring = math.sqrt(max(0.0, 1.0 - z * z))
        az = golden * k
        unit.append([ring * math.cos(az), ring * math.sin(az), z])
    unit = np.array(unit)
    starts = [_start_state(kind, (diameter / 2.0) * unit[k], -(diameter / 2.0) * unit[k]) for k in range(robots)]
    goals = [-((diameter / 2.0) * unit[k]) for k in range(robots)]
    return Problem(kind, np.array(starts), np.array(goals), robot_radius=robot_radius,
                   name=f"antipodal-sphere-{KIND_NAMES[kind]}-n{robots}", **kw)


def random_square(robots: int, diameter: float, seed: int, kind: int = HOLO2D, robot_radius: float = 0.1,
                  min_separation: float | None = None, **kw) -> Problem:
    """scenario.cpp:199-255: starts then goals rejection-sampled uniformly in a
    D×D square (mt19937_64(mix_seed(seed, 0x5c3a))).  `min_separation`
    defaults to the reference's 2·R_a; BASELINE C5 asks for 1 m."""
    eng = MT19937_64(mix_seed(seed, 0x5C3A))
    min_sep = 2.0 * robot_radius if min_separation is None else min_separation

    def sample(what):
        pos = np.zeros((robots, 2))
        for k in range(robots):
            rej = 0
            while True:
                cand = np.array([eng.uniform(-diameter / 2, diameter / 2), eng.uniform(-diameter / 2, diameter / 2)])
                if all(np.linalg.norm(cand - pos[l]) > min_sep for l in range(k)):
                    pos[k] = cand
                    break
                rej += 1
                if rej >= MAX_REJECTIONS:
                    raise ValueError(f"random_square: could not place {what}; workspace too dense")
        return pos

    sp = sample("starts")
    gp = sample("goals")
    starts = np.array([_start_state(kind, sp[k], gp[k]) for k in range(robots)])
    return Problem(kind, starts, gp, robot_radius=robot_radius,
                   name=f"random-square-{KIND_NAMES[kind]}-n{robots}-s{seed}", **kw)


def random_obstacles(problem: Problem, count: int, seed: int, lo: float, hi: float, r_lo: float, r_hi: float,
                     tag: int = 0x0B57) -> Problem:
    """Seeded circular obstacles (builder-defined): centre
    uniform in [lo,hi]^pdim then radius uniform in [r_lo,r_hi], rejected when
    the inflated obstacle touches any start or goal — the clearance test of
    validate_scenario (scenario.cpp:96-106)."""
    eng = MT19937_64(mix_seed(seed, tag))
    pd = problem.pdim
    centers, radii = [], []
    while len(centers) < count:
        rej = 0
        while True:
            c = np.array([eng.uniform(lo, hi) for _ in range(pd)])
            r = eng.uniform(r_lo, r_hi)
            clear = r + problem.robot_radius
            ok = all(np.linalg.norm(problem.starts[k, :pd] - c) > clear and np.linalg.norm(problem.goals[k] - c) > clear
                     for k in range(problem.robots))
            if ok:
                centers.append(c)
                radii.append(r)
                break
            rej += 1
            if rej >= MAX_REJECTIONS:
                raise ValueError("random_obstacles: could not place obstacle")
    out = replace(problem, obs_centers=np.array(centers), obs_radii=np.array(radii))
    out.name = problem.name + f"-obs{count}"
    return out


def cube_corners(edge: float, kind: int = HOLO3D_VEL, robot_radius: float = 0.25, **kw) -> Problem:
    """BASELINE C4: the 8 corners of an edge-length cube, goal = opposite corner."""
    h = edge / 2.0
    pos = np.array([[sx * h, sy * h, sz * h] for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)])
    starts = np.array([_start_state(kind, p, -p) for p in pos])
    return Problem(kind, starts, -pos, robot_radius=robot_radius, name=f"cube-corners-{KIND_NAMES[kind]}", **kw)


def validate(problem: Problem) -> None:
    """validate_scenario (scenario.cpp:46-108) for any model kind."""
    p, R, pd = problem, problem.robots, problem.pdim
    if R < 1:
        raise ValueError("scenario: needs at least one robot")
    if not (np.isfinite(p.starts).all() and np.isfinite(p.goals).all()):
        raise ValueError("scenario: non-finite start or goal")
    min_sep = 2.0 * p.robot_radius
    for k in range(R):
        for l in range(k + 1, R):
            if np.linalg.norm(p.starts[k, :pd] - p.starts[l, :pd]) <= min_sep:
                raise ValueError(f"scenario: robots {k} and {l} start within 2*R_a")
            if np.linalg.norm(p.goals[k] - p.goals[l]) <= min_sep:
                raise ValueError(f"scenario: goals of robots {k} and {l} lie within 2*R_a")
        if np.linalg.norm(p.starts[k, :pd] - p.goals[k]) <= 0.0:
            raise ValueError(f"scenario: robot {k} starts exactly on its goal (degenerate)")
    for o in range(len(p.obs_radii)):
        clear = p.obs_radii[o] + p.robot_radius
        for k in range(R):
            if np.linalg.norm(p.starts[k, :pd] - p.obs_centers[o]) <= clear:
                raise ValueError(f"scenario: start of robot {k} lies inside inflated obstacle {o}")
            if np.linalg.norm(p.goals[k] - p.obs_centers[o]) <= clear:
                raise ValueError(f"scenario: goal of robot {k} lies inside inflated obstacle {o}")


# ------------------------------------------------------------ BASELINE configs
@dataclass
class RunConfig:
    problem: Problem
    samples: int       # BASELINE "N samples/step" = reference DenoiserConfig::batch (M)
    steps: int         # denoising steps per iteration
    iterations: int
    name: str
    lam: float = 0.1
    alpha_bar_final: float = 0.05
    seed: int = 0


def baseline_config(index: int) -> RunConfig:
    """BASELINE.json configs[index-1] (1-based, C1..C5)."""
    if index == 1:
        p = antipodal_circle(4, 8.0, HOLO2D_VEL, robot_radius=0.25, horizon=64, lower=[-1, -1], upper=[1, 1])
        return RunConfig(p, 1024, 100, 1, "C1 holo2d-vel R4 T64 N1024")
    if index == 2:
        p = antipodal_circle(16, 12.0, HOLO2D_VEL, robot_radius=0.25, horizon=128, lower=[-1, -1], upper=[1, 1])
        p = random_obstacles(p, 8, 0, -4.0, 4.0, 0.3, 0.8)
        return RunConfig(p, 8192, 100, 5, "C2 holo2d-vel R16 T128 N8192 O8")
    if index == 3:
        p = antipodal_circle(8, 10.0, UNICYCLE, robot_radius=0.3, horizon=128,
                             lower=[-1.0, -math.pi / 2], upper=[1.0, math.pi / 2])
        return RunConfig(p, 16384, 100, 3, "C3 unicycle R8 T128 N16384")
    if index == 4:
        p = cube_corners(6.0, HOLO3D_VEL, robot_radius=0.25, horizon=128, lower=[-1, -1, -1], upper=[1, 1, 1])
        return RunConfig(p, 16384, 100, 3, "C4 holo3d-vel R8 T128 N16384")
    if index == 5:
        p = random_square(64, 20.0, 0, HOLO2D_VEL, robot_radius=0.2, min_separation=1.0, horizon=256,
                          lower=[-1, -1], upper=[1, 1])
        p = random_obstacles(p, 16, 0, -10.0, 10.0, 0.3, 1.0)
        return RunConfig(p, 262144, 100, 1, "C5 holo2d-vel R64 T256 N262144 O16")
    raise ValueError(f"no BASELINE config {index}")

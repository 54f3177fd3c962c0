"""Benchmark / parity workloads of SURVEY.md §8.0 as configuration texts.

Each workload is a problem definition in the reference's `key = value;` format
(config.cpp:93-171), so the same text drives the engine and the reference's
CPU path (oracle/_ref). Sizes are the reference's own formulas (grid.cpp:34-35,
noise.cpp:141-162, abstraction.cpp:16-48):

  C1   robot reach-avoid, T=8               1,681 states  8,154,531 rows  R=169
  C2a  vehicle3 (bundled), matrix           12,789       319,725         R=27
  C2b  vehicle3, eta/4, matrix, 1 B200      741,393      18,534,825      R=729   (108 GB)
  C3*  room5 normal / uniform / exp / beta  7,776        279,936         R=32/243/243/7776
  C4   7-cell traffic ring, gamma 1e-4      4,782,969    19,131,876      R=78,125 (OFA)
  C4p  traffic5 (bundled), OFA              17,210,368   68,841,472      R=16,807 (OFA)
  C5   BMW 320i 7-d reach-avoid, OFA        157,500      3,937,500       R=7,000
"""
from __future__ import annotations


def _grid(prefix, lb, ub, eta):
    f = lambda v: "{" + ", ".join(repr(float(x)) for x in v) + "}"  # noqa: E731
    return [f"{prefix}.dim = {len(lb)};", f"{prefix}.lb = {f(lb)};", f"{prefix}.ub = {f(ub)};",
            f"{prefix}.eta = {f(eta)};"]


def _vec(v):
    return "{" + ", ".join(repr(float(x)) for x in v) + "}"


def vehicle3(eta=(0.5, 0.5, 0.25), T=32, mode="matrix"):
    """3-d kinematic vehicle parking (C2a; C2b with eta/4)."""
    L = _grid("states", (0, 0, -3.5), (10, 10, 3.5), eta)
    L += _grid("inputs", (-1, -1.5), (1, 1.5), (0.5, 0.75))
    L += ["constants.tau = 0.3;",
          "dynamics.x0 = x0 + tau*u0*cos(x2);",
          "dynamics.x1 = x1 + tau*u0*sin(x2);",
          "dynamics.x2 = x2 + tau*u1;",
          "noise.type = normal;", "noise.sigma = {0.1, 0.1, 0.05};", "noise.mode = additive;",
          "noise.cutting_probability = 0.001;",
          "spec.type = reach-avoid;", f"spec.time_steps = {T};",
          "target.lb = {8.0, 0.0, -3.5};", "target.ub = {10.0, 2.0, 3.5};",
          "avoid.lb = {4.0, 4.0, -3.5};", "avoid.ub = {6.0, 6.0, 3.5};",
          f"exec.mode = {mode};"]
    return "\n".join(L) + "\n"


def bmw7(T=32, mode="ofa", eta=(4.0, 4.0, 0.2, 1.0, 0.1, 0.2, 0.02), ueta=(0.2, 2.0)):
    """7-d single-track BMW 320i parking (C5), piecewise in the heading velocity x3."""
    L = _grid("states", (-10, -10, -0.4, -2, -0.3, -0.4, -0.04), (10, 10, 0.4, 2, 0.3, 0.4, 0.04), eta)
    L += _grid("inputs", (-0.4, -4.0), (0.4, 4.0), ueta)
    consts = dict(tau=0.1, lwb=2.5789, m=1093.3, mu=1.0489, lf=1.156, lr=1.422, hcg=0.6137, iz=1791.6,
                  csf=20.89, csr=20.89, g=9.81)
    L += [f"constants.{k} = {v!r};" for k, v in consts.items()]
    slow = "abs(x3) < 0.1"
    fz = "(g*lr - u1*hcg)"   # front axle load factor
    rz = "(g*lf + u1*hcg)"   # rear axle load factor
    L += [
        f"dynamics.x0 = x0 + tau*ite({slow}, x3*cos(x4), x3*cos(x4 + x6));",
        f"dynamics.x1 = x1 + tau*ite({slow}, x3*sin(x4), x3*sin(x4 + x6));",
        "dynamics.x2 = x2 + tau*u0;",
        "dynamics.x3 = x3 + tau*u1;",
        f"dynamics.x4 = x4 + tau*ite({slow}, (x3/lwb)*tan(x2), x5);",
        f"dynamics.x5 = x5 + tau*ite({slow}, (u1/lwb)*tan(x2) + (x3/(lwb*cos(x2)^2))*u0, "
        f"(mu*m/(iz*(lr + lf)))*(lf*csf*{fz}*x2 + (lr*csr*{rz} - lf*csf*{fz})*x6 - "
        f"(lf^2*csf*{fz} + lr^2*csr*{rz})*(x5/x3)));",
        f"dynamics.x6 = x6 + tau*ite({slow}, 0, (mu/(x3*(lr + lf)))*(csf*{fz}*x2 + "
        f"(csr*{rz} + csf*{fz})*x6 - (lf*csf*{fz} - lr*csr*{rz})*(x5/x3)) - x5);",
    ]
    L += ["noise.type = normal;", "noise.sigma = {0.25, 0.25, 0.2, 0.1, 0.2, 0.2, 0.2};",
          "noise.mode = additive;", "noise.cutting_probability = 0.001;",
          "spec.type = reach-avoid;", f"spec.time_steps = {T};",
          "target.lb = {-1.5, 0.0, -0.4, -2.0, -0.3, -0.4, -0.04};",
          "target.ub = {0.0, 1.5, 0.4, 2.0, 0.3, 0.4, 0.04};",
          "avoid.lb = {-1.5, -0.5, -0.4, -2.0, -0.3, -0.4, -0.04};",
          "avoid.ub = {0.0, 0.0, 0.4, 2.0, 0.3, 0.4, 0.04};",
          f"exec.mode = {mode};"]
    return "\n".join(L) + "\n"


def robot_reachavoid(T=8, mode="ofa"):
    """2-d robot reach-avoid (C1), input pitch 0.1, disturbance grid of 11."""
    L = _grid("states", (-10, -10), (10, 10), (0.5, 0.5))
    L += _grid("inputs", (-1, -1), (1, 1), (0.1, 0.1))
    L += _grid("disturbances", (-1.0,), (1.0,), (0.2,))
    L += ["constants.tau = 10.0;",
          "dynamics.x0 = x0 + tau*u0*cos(u1) + w0;",
          "dynamics.x1 = x1 + tau*u1*sin(u1) + w0;",
          "noise.type = normal;", "noise.sigma = {0.8660254037844386, 0.8660254037844386};",
          "noise.cutting_probability = 0.001;",
          "spec.type = reach-avoid;", f"spec.time_steps = {T};",
          "target.lb = {5.0, 5.0};", "target.ub = {7.0, 7.0};",
          "avoid.lb = {-2.0, -2.0};", "avoid.ub = {2.0, 2.0};", f"exec.mode = {mode};"]
    return "\n".join(L) + "\n"


def traffic_ring(cells=7, eta=1.25, gamma=1e-4, T=7, mode="ofa", ub=10.0):
    """Traffic ring in traffic5's pattern (C4 for 7 cells: x0 fed by the last cell
    and entry u0, x2 by entry u1, odd cells 0.39 decay, the rest 0.64)."""
    n = cells
    L = _grid("states", [0.0] * n, [ub] * n, [eta] * n)
    L += _grid("inputs", (0.0, 0.0), (1.0, 1.0), (1.0, 1.0))
    for i in range(n):
        keep = "0.39" if i % 2 == 1 else "0.64"
        prev = (i - 1) % n
        e = f"{keep}*x{i} + 0.36*x{prev}"
        if i == 0:
            e += " + 6*u0"
        if i == 2:
            e += " + 8*u1"
        L.append(f"dynamics.x{i} = {e};")
    L += ["noise.type = normal;", "noise.sigma = " + _vec([0.7] * n) + ";",
          f"noise.cutting_probability = {gamma!r};",
          "spec.type = safety;", f"spec.time_steps = {T};", f"exec.mode = {mode};"]
    return "\n".join(L) + "\n"


def room5(noise="normal", T=8, mode="matrix"):
    """5-room temperature ring (C3n/u/e/b)."""
    L = _grid("states", [19.0] * 5, [21.0] * 5, [0.4] * 5)
    L += _grid("inputs", (0.0, 0.0), (1.0, 1.0), (0.2, 0.2))
    L += ["constants.ab = 0.378;", "constants.gh = 0.05;", "constants.ghth = 2.5;", "constants.ec = 0.3;",
          "constants.bte = 0.022;",
          "dynamics.x0 = (ab - gh*u0)*x0 + ghth*u0 + ec*(x4 + x1) - bte;",
          "dynamics.x1 = ab*x1 + ec*(x0 + x2) - bte;",
          "dynamics.x2 = (ab - gh*u1)*x2 + ghth*u1 + ec*(x1 + x3) - bte;",
          "dynamics.x3 = ab*x3 + ec*(x2 + x4) - bte;",
          "dynamics.x4 = ab*x4 + ec*(x3 + x0) - bte;"]
    L += {"normal": ["noise.type = normal;", "noise.sigma = " + _vec([0.01] * 5) + ";"],
          "uniform": ["noise.type = uniform;", "noise.a = " + _vec([-0.2] * 5) + ";",
                      "noise.b = " + _vec([0.2] * 5) + ";"],
          "exponential": ["noise.type = exponential;", "noise.rate = " + _vec([100.0] * 5) + ";"],
          "beta": ["noise.type = beta;", "noise.alpha = " + _vec([2.0] * 5) + ";",
                   "noise.beta = " + _vec([5.0] * 5) + ";"]}[noise]
    L += ["noise.cutting_probability = 0.001;", "spec.type = safety;", f"spec.time_steps = {T};",
          f"exec.mode = {mode};"]
    return "\n".join(L) + "\n"


WORKLOADS = {
    "C1": lambda: robot_reachavoid(T=8, mode="matrix"),
    "C2a": lambda: vehicle3(mode="matrix"),
    "C2b": lambda: vehicle3(eta=(0.125, 0.125, 0.0625), mode="matrix"),
    "C3n": lambda: room5("normal"),
    "C3u": lambda: room5("uniform"),
    "C3e": lambda: room5("exponential"),
    "C3b": lambda: room5("beta", mode="ofa"),
    "C4": lambda: traffic_ring(7, 1.25, 1e-4, 7, "ofa"),
    "C4p": lambda: traffic_ring(5, 0.37, 0.02, 7, "ofa"),
    "C5": lambda: bmw7(T=32, mode="ofa"),
}

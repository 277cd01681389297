"""Problem specs and the BASELINE.json workload configs C1..C5.

A `Problem` mirrors the reference `ProblemSpec` (proj/include/hdg/problems.hpp:15-22):
coefficients kappa and c, source f, exact u and flux q = -kappa grad u, and the
boundary classifier used with generated box meshes. Fields are expression
strings compiled by `fields.compile_field` into device-evaluable programs.

The reference registry (proj/src/problems.cpp:52-141) holds paper-sine, poly-k and
constant; C1..C5 are builder-defined per SURVEY.md §8(d) (synthetic inputs with the
BASELINE.json shapes — there is no public dataset for this path).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from .fields import FieldProgram, compile_field


@dataclass
class Problem:
    name: str
    kappa: str
    c: str
    f: str
    u: str
    q: Tuple[str, str, str]
    bc: str = "dirichlet_top_bottom"  # all_dirichlet | dirichlet_top_bottom | dirichlet_x

    def program(self, which: str) -> FieldProgram:
        if which in ("qx", "qy", "qz"):
            return compile_field(self.q["xyz".index(which[1])])
        return compile_field(getattr(self, which))


# problems.cpp:52-87
PAPER_SINE = Problem(
    name="paper-sine",
    kappa="2 + sin(x)*sin(y)*sin(z)",
    c="1 + 0.5*(x*x + y*y + z*z)",
    u="sin(x*y*z)",
    q=("-(2 + sin(x)*sin(y)*sin(z))*y*z*cos(x*y*z)",
       "-(2 + sin(x)*sin(y)*sin(z))*x*z*cos(x*y*z)",
       "-(2 + sin(x)*sin(y)*sin(z))*x*y*cos(x*y*z)"),
    f=("-((cos(x)*sin(y)*sin(z)*y*z + sin(x)*cos(y)*sin(z)*x*z + sin(x)*sin(y)*cos(z)*x*y)"
       "*cos(x*y*z)) - (2 + sin(x)*sin(y)*sin(z))*(-(y*y*z*z + x*x*z*z + x*x*y*y)*sin(x*y*z))"
       " + (1 + 0.5*(x*x + y*y + z*z))*sin(x*y*z)"),
    bc="dirichlet_top_bottom",
)

# problems.cpp:118-126
CONSTANT = Problem(name="constant", kappa="1", c="1", u="1", f="1", q=("0", "0", "0"))


def _mono(a: int, b: int, c: int) -> str:
    parts = ["x"] * a + ["y"] * b + ["z"] * c
    return "*".join(parts) if parts else "1"


def poly_k(degree: int, terms: Sequence[Tuple[int, int, int, float]]) -> Problem:
    """problems.cpp:89-116 given the monomial list (coef from std::mt19937(12345+k))."""
    kap, cc = 2.0, 1.0

    def poly(ts):
        return " + ".join(f"({coef!r})*{_mono(a, b, c)}" for a, b, c, coef in ts) or "0"

    def deriv(ts, axis):
        out = []
        for a, b, c, coef in ts:
            e = (a, b, c)[axis]
            if e == 0:
                continue
            n = [a, b, c]
            n[axis] -= 1
            out.append((n[0], n[1], n[2], coef * e))
        return out

    dx, dy, dz = (deriv(terms, i) for i in range(3))
    lap = deriv(dx, 0) + deriv(dy, 1) + deriv(dz, 2)
    f_terms = [(a, b, c, cc * co) for a, b, c, co in terms] + [(a, b, c, -kap * co) for a, b, c, co in lap]
    return Problem(
        name=f"poly-{degree}", kappa=repr(kap), c=repr(cc), u=poly(terms),
        q=(f"-{kap!r}*({poly(dx)})", f"-{kap!r}*({poly(dy)})", f"-{kap!r}*({poly(dz)})"),
        f=poly(f_terms), bc="dirichlet_top_bottom")


# ----------------------------------------------------------- BASELINE configs
_C2_KAPPA = "1 + 0.5*sin(2*pi*x)*cos(2*pi*y)"
_C2_U = "exp(x + y)*sin(pi*z)"
# q = -kappa grad u; f = div q + c u = u*(-pi*cos(2*pi*(x+y)) - kappa*(2 - pi^2) + c)
_C2 = Problem(
    name="c2-varcoef",
    kappa=_C2_KAPPA,
    c="1 + x*y*z",
    u=_C2_U,
    q=(f"-({_C2_KAPPA})*exp(x + y)*sin(pi*z)",
       f"-({_C2_KAPPA})*exp(x + y)*sin(pi*z)",
       f"-({_C2_KAPPA})*pi*exp(x + y)*cos(pi*z)"),
    f=f"exp(x + y)*sin(pi*z)*(-pi*cos(2*pi*(x + y)) - ({_C2_KAPPA})*(2 - pi*pi) + 1 + x*y*z)",
    bc="dirichlet_x",
)
_C1_U = "sin(pi*x)*sin(pi*y)*sin(pi*z)"
_C1 = Problem(
    name="c1-sine", kappa="1", c="1", u=_C1_U,
    q=("-pi*cos(pi*x)*sin(pi*y)*sin(pi*z)", "-pi*sin(pi*x)*cos(pi*y)*sin(pi*z)",
       "-pi*sin(pi*x)*sin(pi*y)*cos(pi*z)"),
    f=f"(3*pi*pi + 1)*{_C1_U}", bc="all_dirichlet")
# C3: kappa ratio 1:100 across z = 0.5 (element-aligned), c = 0, f = sin sin sin,
# u_D = 0, g = 0; no exact solution (parity + throughput config).
_C3 = Problem(
    name="c3-jump", kappa="(1 + 0.25*sin(2*pi*x)*sin(2*pi*y))*(100 - 99*lt(z, 0.5))", c="0",
    u="sin(pi*x)*sin(pi*y)*sin(pi*z)", q=("0", "0", "0"),
    f="sin(pi*x)*sin(pi*y)*sin(pi*z)", bc="dirichlet_top_bottom")
_C4_U = "x*y*z*(1 - x)*(1 - y)*(1 - z)"
_C4 = Problem(
    name="c4-convdiff", kappa="0.01", c="1", u=_C4_U,
    q=("-0.01*y*z*(1 - y)*(1 - z)*(1 - 2*x)", "-0.01*x*z*(1 - x)*(1 - z)*(1 - 2*y)",
       "-0.01*x*y*(1 - x)*(1 - y)*(1 - 2*z)"),
    f=("0.02*(y*z*(1 - y)*(1 - z) + x*z*(1 - x)*(1 - z) + x*y*(1 - x)*(1 - y))"
       f" + {_C4_U}"),
    bc="all_dirichlet")
C4_BETA = ("sin(pi*y)", "cos(pi*x)", "0.5")


@dataclass
class Config:
    """One BASELINE.json workload: mesh, degree, stabilisation and problem."""
    name: str
    n: int                       # cells per axis of the Kuhn box
    k: int
    problem: Problem
    tau: float = 1.0             # constant tau (C4 overrides with the upwind rule)
    perturb: float = 0.0         # interior-vertex jitter as a fraction of h (C3)
    seed: int = 1305
    upwind_beta: Optional[Tuple[str, str, str]] = None  # C4: tau = 1 + |beta(x_e).nu|
    postprocess: bool = False    # C5: P_{k+1} postprocess in the step
    note: str = ""

    @property
    def nelt(self) -> int:
        return 6 * self.n ** 3

    @property
    def quad_degree(self) -> int:  # study.cpp:13-14
        return 2 * self.k + 2


CONFIGS: Dict[str, Config] = {
    "C1": Config("C1", 8, 1, _C1, note="k=1, 8^3 Kuhn, kappa=c=tau=1, all Dirichlet"),
    "C2": Config("C2", 32, 3, _C2, note="k=3, 32^3 Kuhn, variable kappa/c, Dirichlet x=0,1"),
    "C3": Config("C3", 24, 5, _C3, tau=24.0, perturb=0.15,
                 note="k=5, 24^3 perturbed, kappa jump 1:100, c=0, tau=1/h"),
    "C4": Config("C4", 48, 2, _C4, upwind_beta=C4_BETA,
                 note="k=2, 48^3, conv-diff block, tau=1+|beta.nu|"),
    "C5": Config("C5", 64, 3, _C2, postprocess=True, note="k=3 + P4, 64^3, C2 fields"),
}


def scaled(cfg: Config, n: int) -> Config:
    """The same config on an n^3 box (parity tests run shrunken meshes)."""
    import dataclasses
    out = dataclasses.replace(cfg, n=n)
    if cfg.perturb:
        out = dataclasses.replace(out, tau=float(n))  # tau = 1/h keeps its meaning
    return out

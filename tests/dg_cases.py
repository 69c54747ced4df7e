"""DG test cases shared by the fixture generator (tests/golden/make_golden_dg.py,
run against the reference) and the GPU parity tests (tests/test_gpu_dg.py).
Expressions are numpy callables taking x=, y=, t= keywords, as the
reference's parsed expressions do (solvers.py:79-89)."""
import numpy as np


def const(v):
    return lambda x, y, t=0.0: v + 0.0 * x


WALLS = {name: {"type": "rigid_wall"} for name in ("south", "east", "north", "west")}
PERIODIC_BOX = {"south": {"type": "periodic", "pair": "north"},
                "north": {"type": "periodic", "pair": "south"},
                "west": {"type": "periodic", "pair": "east"},
                "east": {"type": "periodic", "pair": "west"}}
MIXED = {"west": {"type": "periodic", "pair": "east"},
         "east": {"type": "periodic", "pair": "west"},
         "south": {"type": "farfield"},
         "north": {"type": "dirichlet",
                   "value": lambda x, y, t=0.0: 0.1 * np.sin(np.pi * x) * (1.0 + t)}}

BASE_VARIABLE = {"ux": lambda x, y, t=0.0: 0.3 * y, "uy": lambda x, y, t=0.0: -0.2 * x,
                 "rho": lambda x, y, t=0.0: 1.2 + 0.1 * x,
                 "c2": lambda x, y, t=0.0: 1.5 + 0.2 * y}
BASE_UNIFORM = {"ux": const(0.4), "uy": const(-0.2), "rho": const(1.3), "c2": const(2.0)}
INITIAL = {"p": lambda x, y, t=0.0: np.exp(-8 * ((x - 0.4) ** 2 + (y - 0.5) ** 2)),
           "ux": lambda x, y, t=0.0: 0.2 * np.sin(np.pi * x),
           "uy": lambda x, y, t=0.0: -0.1 * np.cos(np.pi * y)}
SOURCE_P = {"p": lambda x, y, t=0.0: np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y) * (1.0 + t)}

CASES = {
    "walls": {"mesh": (3, 3), "P": 4, "bcs": WALLS, "primitives": True,
              "ape": [{"base": BASE_VARIABLE, "initial": INITIAL, "riemann": "upwind"},
                      {"base": BASE_VARIABLE, "initial": INITIAL, "riemann": "laxfriedrichs"}]},
    "periodic": {"mesh": (4, 4), "P": 5, "bcs": PERIODIC_BOX, "primitives": True,
                 "ape": [{"base": BASE_UNIFORM, "initial": INITIAL, "riemann": "upwind",
                          "sources": SOURCE_P, "t": 0.25}],
                 "advection": [{"velocity": (const(1.0), lambda x, y, t=0.0: 0.5 - 0.3 * x)}]},
    "mixed": {"mesh": (5, 2), "P": 3, "bcs": MIXED, "primitives": True,
              "ape": [{"base": BASE_VARIABLE, "initial": INITIAL, "riemann": "upwind", "t": 0.5}],
              "advection": [{"velocity": (const(0.7), const(0.4)), "t": 0.5}]},
}

"""B200-native partial-fraction matrix functions (hot path of arXiv 2210.03714).

Host-side method tables (exact) live in `methods`; the device path is reached through the C ABI
(include/pf_b200.h) via `api`. Importing `api` loads the CUDA engine and fails loudly if it is
missing -- there is no CPU fallback.
"""
from .errors import Errc, PfError  # noqa: F401
from .methods import (PLAIN, RESIDUAL, THETA_U53, FractionMethod, FunctionId, catalog, catalog_names,  # noqa: F401
                      pair_method, same_shift_method, theta, to_double_nearest, to_plain_form, to_residual_form)


def __getattr__(name):
    # lazy: `import paper_2210_03714_b200` works without a GPU (host tables, build, tests);
    # touching the device API loads the engine.
    if name in ("api", "eval_dense", "expm", "expm_phi1", "cossin", "solve_shifted", "one_norm", "gemm",
                "EvalOptions", "Engine", "engine"):
        import importlib

        api = importlib.import_module(__name__ + ".api")
        return api if name == "api" else getattr(api, name)
    raise AttributeError(name)

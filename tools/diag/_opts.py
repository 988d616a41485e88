"""Diagnostics helper: apply LSRN_OPT_<NAME>=value environment settings of the TOOL's
process to a context through lsrn_ctx_set_option (the library itself reads no
environment variables)."""
import os


def apply_env_options(ctx):
    from paper_1109_5981_b200 import lsrn
    used = {}
    for k, v in os.environ.items():
        if k.startswith("LSRN_OPT_"):
            name = k[len("LSRN_OPT_"):].lower()
            if name in lsrn.OPTIONS:
                ctx.set_option(name, v if name == "svd" and not v.lstrip("-").isdigit() else int(v))
                used[name] = v
    return used

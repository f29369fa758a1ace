"""Build libdbag.so variants with different -D tuning macros into
paper_1708_07954_b200/_variants/<name>.so (A/B timing via DBAG_LIB=...)."""
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_07954_b200 import build as b  # noqa: E402

# Each entry toggles one knob of the current kernels away from its default
# (DESIGN.md §4 records the measured outcome of each); "cur" is the default.
VARIANTS = {
    "cur": [],
    # EXACT K1 (dbag_exact.cu)
    "exact_t96": ["-DDBAG_K1E_THREADS=96"],
    "exact_t64": ["-DDBAG_K1E_THREADS=64"],
    "exact_t128": ["-DDBAG_K1E_THREADS=128"],
    "exact_t384": ["-DDBAG_K1E_THREADS=384"],
    "exact_nosync": ["-DDBAG_K1E_SYNC=0"],
    "exact_sync2": ["-DDBAG_K1E_SYNC=2"],
    "exact_syncg2": ["-DDBAG_K1E_SYNCGROUP=2"],
    "exact_syncg2_t256": ["-DDBAG_K1E_SYNCGROUP=2", "-DDBAG_K1E_THREADS=256"],
    "exact_batch0": ["-DDBAG_K1E_BATCH=0", "-DDBAG_K1E_LEAN=0"],
    "exact_batch32": ["-DDBAG_K1E_BATCH=32"],
    "exact_batch128": ["-DDBAG_K1E_BATCH=128"],
    "exact_lean0": ["-DDBAG_K1E_LEAN=0"],
    "exact_prefetch": ["-DDBAG_K1E_PREFETCH=1", "-DDBAG_K1E_LEAN=0"],
    "exact_mdiv0": ["-DDBAG_K1E_MDIV=0"],
    "exact_mdsolve0": ["-DDBAG_K1E_MDSOLVE=0"],
    "exact_mdtgt0": ["-DDBAG_K1E_MDTGT=0"],
    "exact_roll0": ["-DDBAG_K1E_ROLLTGT=0", "-DDBAG_K1E_ROLLTRIG=0"],
    "exact_rolltrig0": ["-DDBAG_K1E_ROLLTRIG=0"],
    "exact_rcpfast0": ["-DDBAG_K1E_RCPFAST=0"],
    "exact_sinconst0": ["-DDBAG_SINCOS_CONST=0"],
    "exact_finmax0": ["-DDBAG_K1E_FINMAX=0"],
    "exact_jacinline0": ["-DDBAG_K1E_JACINLINE=0"],
    "exact_lean2_0": ["-DDBAG_K1E_LEAN2=0"],
    "exact_lean3_0": ["-DDBAG_K1E_LEAN3=0"],
    "exact_hubp": ["-DDBAG_K1E_HUBP=1"],
    "exact_hub_minb2": ["-DDBAG_K1E_HUB_MINB=2"],
    "k2_group0": ["-DDBAG_K2E_GROUP=0"],
    "k2_g4": ["-DDBAG_K2E_G=4"],
    "k2_g2": ["-DDBAG_K2E_G=2"],
    "k2_g16": ["-DDBAG_K2E_G=16"],
    "exact_hub_minb4": ["-DDBAG_K1E_HUB_MINB=4"],
    # FAST K1 (dbag_local.cuh via dbag_capi.cu)
    "fast_v2": ["-DDBAG_FAST_V4=0", "-DDBAG_FAST_V3=0"],
    "fast_v3": ["-DDBAG_FAST_V4=0"],
    "fast_sync": ["-DDBAG_K1_SYNC=1"],
    "fast_minb3": ["-DDBAG_K1_MINB=3"],
    "fast_hub_minb2": ["-DDBAG_K1_HUB_MINB=2"],
    "fast_hub_minb3": ["-DDBAG_K1_HUB_MINB=3"],
    # generalized blocks (dbag_blocks.cu)
    "gen_colmajor": ["-DDBAG_GEN_COLMAJOR=1"],
    "gen_parpiv0": ["-DDBAG_GEN_PARPIV=0"],
    "gen_warp128": ["-DDBAG_WARP_BLOCK_MAX_DIM=128", "-DDBAG_GEN_X"],
    "gen_warp24": ["-DDBAG_WARP_BLOCK_MAX_DIM=24", "-DDBAG_GEN_X"],
}


def main(names):
    out = os.path.join(b.HERE, "_variants")
    os.makedirs(out, exist_ok=True)
    saved = b.LIB
    for n in names or VARIANTS:
        b.LIB = os.path.join(out, n + ".so")
        fl = VARIANTS[n]
        fast = any("DBAG_FAST" in f or "DBAG_K1_" in f for f in fl)
        gen = any("DBAG_GEN" in f for f in fl)
        b.build(force=True, extra=fl, only=["dbag_blocks.cu" if gen else
                                            "dbag_capi.cu" if fast else "dbag_exact.cu"])
        print("built", b.LIB)
    b.LIB = saved


if __name__ == "__main__":
    main(sys.argv[1:])

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
    # EXACT K1, squared L2 (dbag_exact.cu k_local_gn_exact)
    "exact_t96": ["-DDBAG_K1E_THREADS=96"],
    "exact_t192": ["-DDBAG_K1E_THREADS=192"],
    "exact_batch32": ["-DDBAG_K1E_BATCH=32"],
    "exact_batch128": ["-DDBAG_K1E_BATCH=128"],
    "exact_effort_off": ["-DDBAG_EFFORT_MAX_L=0"],
    # EXACT K1, Huber (dbag_exact.cu k_local_huber_pool): pool size / CTAs per SM
    "hub_ls1": ["-DDBAG_HUB_LS=1"],
    "hub_ls3": ["-DDBAG_HUB_LS=3"],
    "hub_ls5": ["-DDBAG_HUB_LS=5"],
    "hub_q40": ["-DDBAG_HUB_Q=40", "-DDBAG_HUB_MINB=12"],
    "hub_q56": ["-DDBAG_HUB_Q=56", "-DDBAG_HUB_MINB=8"],
    "hub_q64": ["-DDBAG_HUB_Q=64", "-DDBAG_HUB_MINB=7"],
    "hub_fixed3": ["-DDBAG_HUB_LS_MIN=1", "-DDBAG_HUB_LS=3"],
    "hub_m20_l8": ["-DDBAG_HUB_LS_MIN=20", "-DDBAG_HUB_LS=8"],
    "k2_minb3": ["-DDBAG_K2E_MINB=3"],
    # K3 exact: the streamed persistent kernel off / ring depth
    "k3_percam": ["-DDBAG_K3_STREAM_MIN_OBS=2000000000"],
    "k3_stream": ["-DDBAG_K3_STREAM_MIN_OBS=1024"],
    "k3s_t768": ["-DDBAG_K3S_THREADS=768"],
    "k3s_t640": ["-DDBAG_K3S_THREADS=640"],
    "k3s_p7": ["-DDBAG_K3S_PROD=7"],
    "k3s_sl0": ["-DDBAG_K3S_SLEEP=0"],
    # K2 exact: lanes per point
    "k2_g4": ["-DDBAG_K2E_G=4"],
    "k2_g8": ["-DDBAG_K2E_G=8"],
    # FAST K1 (dbag_local.cuh via dbag_capi.cu)
    "fast_minb3": ["-DDBAG_K1_MINB=3"],
    # generalized blocks (dbag_blocks.cu)
    "gen_warp128": ["-DDBAG_WARP_BLOCK_MAX_DIM=128", "-DDBAG_GEN_X"],
}


def main(names):
    out = os.path.join(b.HERE, "_variants")
    os.makedirs(out, exist_ok=True)
    saved = b.LIB
    for n in names or VARIANTS:
        b.LIB = os.path.join(out, n + ".so")
        fl = VARIANTS[n]
        fast = any("DBAG_FAST" in f or "DBAG_K1_" in f or "DBAG_EFFORT" in f for f in fl)
        gen = any("DBAG_GEN" in f for f in fl)
        b.build(force=True, extra=fl, only=["dbag_blocks.cu" if gen else
                                            "dbag_capi.cu" if fast else "dbag_exact.cu"])
        print("built", b.LIB)
    b.LIB = saved


if __name__ == "__main__":
    main(sys.argv[1:])

"""Build libdbag.so variants with different -D tuning macros into
paper_1708_07954_b200/_variants/<name>.so (A/B timing via DBAG_LIB=...)."""
import os
import shutil
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_07954_b200 import build as b  # noqa: E402

VARIANTS = {
    "base": [],
    "fast_minb3": ["-DDBAG_K1_MINB=3"],
    "fast_minb4": ["-DDBAG_K1_MINB=4"],
    "exact_minb2": ["-DDBAG_K1E_MINB=2"],
    "exact_minb3": ["-DDBAG_K1E_MINB=3"],
    "exact_minb4": ["-DDBAG_K1E_MINB=4"],
    "jcache0": ["-DDBAG_K1E_JCACHE=0"],
    "jcache1": ["-DDBAG_K1E_JCACHE=1"],
    "smstate0": ["-DDBAG_K1E_SMSTATE=0"],
    "smstate1": ["-DDBAG_K1E_SMSTATE=1"],
    "abl_pivot": ["-DDBAG_ABLATE_PIVOT"],
    "fastpiv0": ["-DDBAG_K1E_FASTPIV=0"],
    "fastpiv1": ["-DDBAG_K1E_FASTPIV=1"],
    "packord0": ["-DDBAG_K1E_PACKORD=0"],
    "mdiv0": ["-DDBAG_K1E_MDIV=0"],
    "mdiv1": ["-DDBAG_K1E_MDIV=1"],
    "cur": [],
    "fsync0": ["-DDBAG_K1_SYNC=0"],
    "split1": ["-DDBAG_K1E_SPLITREFILL=1"],
    "t96": ["-DDBAG_K1E_THREADS=96"],
    "t64": ["-DDBAG_K1E_THREADS=64"],
    "t160": ["-DDBAG_K1E_THREADS=160", "-DDBAG_K1E_MINB=2"],
    "t192": ["-DDBAG_K1E_THREADS=192"],
    "t384": ["-DDBAG_K1E_THREADS=384"],
    "sync2": ["-DDBAG_K1E_SYNC=2"],
    "sync4": ["-DDBAG_K1E_SYNC=4"],
    "rcpfast0": ["-DDBAG_K1E_RCPFAST=0"],
    "lean0": ["-DDBAG_K1E_LEAN=0"],
    "colmajor0": ["-DDBAG_GEN_COLMAJOR=0"],
    "hubp0": ["-DDBAG_K1E_HUBP=0"],
    "fastv2": ["-DDBAG_FAST_V3=0"],
    "batch0": ["-DDBAG_K1E_BATCH=0"],
    "pf0": ["-DDBAG_K1E_PREFETCH=0"],
    "pf0_sync0": ["-DDBAG_K1E_PREFETCH=0", "-DDBAG_K1E_SYNC=0"],
    "batch64": ["-DDBAG_K1E_BATCH=64"],
    "nosync": ["-DDBAG_K1E_SYNC=0"],
    "mdsolve0": ["-DDBAG_K1E_MDSOLVE=0"],
    "mdtgt0": ["-DDBAG_K1E_MDTGT=0"],
    "pivcall0": ["-DDBAG_K1E_PIVCALL=0"],
    "pivcall1": ["-DDBAG_K1E_PIVCALL=1"],
    "sincoscall": ["-DDBAG_SINCOS_CALL=1"],
    "sync128": ["-DDBAG_K1E_SYNC=1"],
    "sync384": ["-DDBAG_K1E_SYNC=1", "-DDBAG_K1E_THREADS=384"],
    "t384": ["-DDBAG_K1E_THREADS=384"],
    "sync128_mdiv1": ["-DDBAG_K1E_SYNC=1", "-DDBAG_K1E_MDIV=1"],
    "unified0": ["-DDBAG_K1E_UNIFIED=0"],
    "unified1": ["-DDBAG_K1E_UNIFIED=1"],
    "unified1_mdiv1": ["-DDBAG_K1E_UNIFIED=1", "-DDBAG_K1E_MDIV=1"],
    "roll0": ["-DDBAG_K1E_ROLLTGT=0", "-DDBAG_K1E_ROLLTRIG=0"],
    "roll1": [],
    "roll1_mdiv1": ["-DDBAG_K1E_MDIV=1"],
    "mdiv0": ["-DDBAG_K1E_MDIV=0"],
    "mdiv1": ["-DDBAG_K1E_MDIV=1"],
    "cur": [],
    "fsync0": ["-DDBAG_K1_SYNC=0"],
    "split1": ["-DDBAG_K1E_SPLITREFILL=1"],
    "t96": ["-DDBAG_K1E_THREADS=96"],
    "t64": ["-DDBAG_K1E_THREADS=64"],
    "t160": ["-DDBAG_K1E_THREADS=160", "-DDBAG_K1E_MINB=2"],
    "t192": ["-DDBAG_K1E_THREADS=192"],
    "t384": ["-DDBAG_K1E_THREADS=384"],
    "sync2": ["-DDBAG_K1E_SYNC=2"],
    "sync4": ["-DDBAG_K1E_SYNC=4"],
    "rcpfast0": ["-DDBAG_K1E_RCPFAST=0"],
    "lean0": ["-DDBAG_K1E_LEAN=0"],
    "colmajor0": ["-DDBAG_GEN_COLMAJOR=0"],
    "hubp0": ["-DDBAG_K1E_HUBP=0"],
    "fastv2": ["-DDBAG_FAST_V3=0"],
    "batch0": ["-DDBAG_K1E_BATCH=0"],
    "pf0": ["-DDBAG_K1E_PREFETCH=0"],
    "pf0_sync0": ["-DDBAG_K1E_PREFETCH=0", "-DDBAG_K1E_SYNC=0"],
    "batch64": ["-DDBAG_K1E_BATCH=64"],
    "nosync": ["-DDBAG_K1E_SYNC=0"],
    "mdsolve0": ["-DDBAG_K1E_MDSOLVE=0"],
    "mdtgt0": ["-DDBAG_K1E_MDTGT=0"],
    "sync256": ["-DDBAG_K1E_SYNC=1", "-DDBAG_K1E_THREADS=64"],
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

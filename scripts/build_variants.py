"""Build tuning variants of libchebld.so into build_variants/ (git-ignored)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_06394_b200 import _build  # noqa: E402

VARIANTS = {
    "s3": ["CHEB_STAGES=3"],
    "s3c3": ["CHEB_STAGES=3", "CHEB_MIN_CTAS=3"],
    "c3": ["CHEB_MIN_CTAS=3"],
    "r1c4": ["CHEB_MIN_CTAS_R1=4"],
    "dec": ["CHEB_DECOUPLE=1"],
    "fam4": ["CHEB_MIN_CTAS_FAM=4"],
    "cap6dec": ["CHEB_CAP_PER_ROW=6", "CHEB_DECOUPLE=1"],
    "cap6": ["CHEB_CAP_PER_ROW=6"],
    "narrow": ["CHEB_WIDE=0"],
    "wide16": ["CHEB_WIDE_MAXK=16"],
    "sus1k": ["CHEB_MBAR_SUSPEND_NS=1000"],
    "sus20k": ["CHEB_MBAR_SUSPEND_NS=20000"],
    "s3sus1k": ["CHEB_STAGES=3", "CHEB_MBAR_SUSPEND_NS=1000"],
    "diag_r1nosync": ["CHEB_DIAG_R1_NOSYNC=1"],  # timing diagnostic: wrong rank-1 moments
    "diag_r1nosync_c4": ["CHEB_DIAG_R1_NOSYNC=1", "CHEB_MIN_CTAS_R1=4"],
    "dec3": ["CHEB_DECOUPLE=1", "CHEB_STAGES=3"],
    "r1": ["CHEB_RPG=1"],
    "r4": ["CHEB_RPG=4"],
    "checked": ["CHEB_CHECKS=1"],
    "resprof": ["CHEB_RES_PROF=1"],
    "rest640": ["CHEB_RES_THREADS=640"],  # resident kernel: 20 warps per SM at 96 registers
    "nocv": ["CHEB_CV_KERNEL=0"],  # step kernels without the compressed-copy path (A/B)
    "resdiag1": ["CHEB_RES_PROF=1", "CHEB_RES_DIAG=1"],  # timing diagnostics: wrong results
    "resdiag2": ["CHEB_RES_PROF=1", "CHEB_RES_DIAG=2"],  # per-CTA phase cycles of the resident kernel (scripts/res_phases.py)
    "u4c4": ["CHEB_NNZ_UNROLL=4", "CHEB_MIN_CTAS=4"],
    "u8c3": ["CHEB_NNZ_UNROLL=8", "CHEB_MIN_CTAS=3"],
    "dbl4": ["CHEB_MIN_CTAS_DBL=4"],
    "dblwc": ["CHEB_DBL_STAGE_WC=1"],
    # 8 probes per lane needs >= 2 rows per lane group at PPL 4, also for the doubling kernels
    "p8c2": ["CHEB_PPL=8", "CHEB_MIN_CTAS=2", "CHEB_MIN_CTAS_DBL=2", "CHEB_RPG_DBL=2", "CHEB_DBL_STAGE_WC=0"],
    "p8u3c3": ["CHEB_PPL=8", "CHEB_NNZ_UNROLL=3", "CHEB_MIN_CTAS=3", "CHEB_MIN_CTAS_DBL=3", "CHEB_RPG_DBL=2",
               "CHEB_DBL_STAGE_WC=0"],
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    root = os.path.join(_build.ROOT, "build_variants")
    os.makedirs(root, exist_ok=True)
    with ThreadPoolExecutor(4) as ex:
        for p in ex.map(lambda n: _build.build(force=True, out=os.path.join(root, f"libchebld_{n}.so"),
                                              defines=VARIANTS[n]), names):
            print(p)

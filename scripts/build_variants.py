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
    "dr2": ["CHEB_RPG_DBL=2"],
    "dwc": ["CHEB_DBL_STAGE_WC=1"],
    "r1": ["CHEB_RPG=1"],
    "r1s3": ["CHEB_RPG=1", "CHEB_STAGES=3"],
    "r4": ["CHEB_RPG=4"],
    "r4c3": ["CHEB_RPG=4", "CHEB_MIN_CTAS=3"],
    "checked": ["CHEB_CHECKS=1"],
    "f_s1": ["CHEB_FUSED_SLACK=1"],
    "f_s2": ["CHEB_FUSED_SLACK=2"],
    "f_s1h": ["CHEB_FUSED_SLACK=1", "CHEB_FUSED_HINTS=1"],
    "f_s2h": ["CHEB_FUSED_SLACK=2", "CHEB_FUSED_HINTS=1"],
    "u4c4": ["CHEB_NNZ_UNROLL=4", "CHEB_MIN_CTAS=4"],
    "u8c3": ["CHEB_NNZ_UNROLL=8", "CHEB_MIN_CTAS=3"],
    "u8c2": ["CHEB_NNZ_UNROLL=8", "CHEB_MIN_CTAS=2"],
    "u6c3": ["CHEB_NNZ_UNROLL=6", "CHEB_MIN_CTAS=3"],
    "u5c4": ["CHEB_NNZ_UNROLL=5", "CHEB_MIN_CTAS=4"],
    "dbl4": ["CHEB_MIN_CTAS_DBL=4"],
    "dblwc": ["CHEB_DBL_STAGE_WC=1"],
    "dbl4u4": ["CHEB_MIN_CTAS_DBL=4", "CHEB_NNZ_UNROLL=4"],
    "fc3": ["CHEB_FUSED_MIN_CTAS=3"],
    "fc3s1": ["CHEB_FUSED_MIN_CTAS=3", "CHEB_FUSED_SLACK=1"],
    "fs1": ["CHEB_FUSED_SLACK=1"],
    "ffence": ["CHEB_FUSED_FENCE=1"],
    "w2": ["CHEB_FUSEDW_STAGES=2"],
    "pf1": ["CHEB_L2_PREFETCH=1"],
    "gs2w": ["CHEB_GS_STAGES=2", "CHEB_GS_LIST=4096"],
    "gs4s": ["CHEB_GS_STAGES=4", "CHEB_GS_LIST=2048"],
    "wc4": ["CHEB_FUSEDW_MIN_CTAS=4"],
    "dr1wc4": ["CHEB_RPG=1", "CHEB_DBL_STAGE_WC=1", "CHEB_MIN_CTAS_DBL=4"],
    "dr1wc3": ["CHEB_RPG=1", "CHEB_DBL_STAGE_WC=1", "CHEB_MIN_CTAS_DBL=3"],
    "dr1c4": ["CHEB_RPG=1", "CHEB_MIN_CTAS_DBL=4"],
    "wc4s2": ["CHEB_FUSEDW_MIN_CTAS=4", "CHEB_FUSEDW_STAGES=2"],
    "w4": ["CHEB_FUSEDW_STAGES=4", "CHEB_FUSEDW_MIN_CTAS=2"],
    # 8 probes per lane needs >= 2 rows per lane group at PPL 4, also for the doubling kernels
    "p8c2": ["CHEB_PPL=8", "CHEB_MIN_CTAS=2", "CHEB_MIN_CTAS_DBL=2", "CHEB_RPG_DBL=2", "CHEB_DBL_STAGE_WC=0"],
    "p8u3c3": ["CHEB_PPL=8", "CHEB_NNZ_UNROLL=3", "CHEB_MIN_CTAS=3", "CHEB_MIN_CTAS_DBL=3", "CHEB_RPG_DBL=2",
               "CHEB_DBL_STAGE_WC=0"],
    "p8u3c2": ["CHEB_PPL=8", "CHEB_NNZ_UNROLL=3", "CHEB_MIN_CTAS=2", "CHEB_MIN_CTAS_DBL=2", "CHEB_RPG_DBL=2",
               "CHEB_DBL_STAGE_WC=0"],
    "p8u5c3": ["CHEB_PPL=8", "CHEB_MIN_CTAS=3", "CHEB_MIN_CTAS_DBL=3", "CHEB_RPG_DBL=2", "CHEB_DBL_STAGE_WC=0"],
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    root = os.path.join(_build.ROOT, "build_variants")
    os.makedirs(root, exist_ok=True)
    with ThreadPoolExecutor(4) as ex:
        for p in ex.map(lambda n: _build.build(force=True, out=os.path.join(root, f"libchebld_{n}.so"),
                                              defines=VARIANTS[n]), names):
            print(p)

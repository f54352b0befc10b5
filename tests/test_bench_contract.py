"""CPU tier: the bench's accounting (SURVEY.md 8(d) algorithmic bytes, the
kernel each BASELINE config dispatches to) -- the numbers the roofline
fractions in every bench line are computed from."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402

N = 100_000_000


def test_c_lp_s_bytes_match_survey_8d():
    # 11N + N/g HBM, 2N(g-1)/g NVLink ingress
    assert bench.algorithmic_bytes("c_lp_s", N, 1) == (12 * N, 0)
    assert bench.algorithmic_bytes("c_lp_s", N, 8) == (11 * N + N // 8, 2 * N * 7 // 8)
    hbm, nvl = bench.algorithmic_bytes("c_lp_s", N, 4)
    assert nvl == 150_000_000 and hbm == 1_125_000_000


def test_c_fp_s_and_d_bytes():
    assert bench.algorithmic_bytes("c_fp_s", 25_000_000, 1) == (0, 0)  # collectives.cpp:49
    assert bench.algorithmic_bytes("c_fp_s", 25_000_000, 8)[1] == 8 * 25_000_000 * 7 // 8
    # D_FP_S ring at g = 8: |N| = 3, 16N HBM, 8N ingress
    assert bench.algorithmic_bytes("d_fp_s", 25_000_000, 8) == (16 * 25_000_000, 8 * 25_000_000)
    assert bench.algorithmic_bytes("codec", 4_000_000, 1) == (40_000_000, 0)


def test_kernel_labels_follow_the_dispatch():
    assert bench.kernel_label("c_lp_s", N, 1).startswith("central_kernel<uint8>")
    assert bench.kernel_label("c_lp_s", N, 2).startswith("central_stag_kernel")
    assert bench.kernel_label("c_lp_s", N, 4).startswith("central_kernel<uint8>")
    assert bench.kernel_label("c_lp_s", 1_000_000, 2).startswith("central_small_kernel<uint8")
    assert bench.kernel_label("c_fp_s", 25_000_000, 4).startswith("central_kernel<identity>")
    assert bench.kernel_label("d_lp_s", 1_000_000, 2).startswith("decent_small_kernel")
    assert bench.kernel_label("d_lp_s", 100_000_000, 2).startswith("decent_kernel<uint8>")

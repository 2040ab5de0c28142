"""Packed-record ADC scan == generic ADC scan (bit-exact ids and float64 distances),
exhaustive and candidate-list modes, with duplicate candidates and exact ties."""

import numpy as np
import pytest
import torch

from paper_1509_05194_b200 import _engine as E

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,K,r", [(8, 256, 100), (4, 16, 7), (1, 4, 3), (8, 2, 50)])
def test_packed_scan_matches_generic(M, K, r):
    g = torch.Generator(device="cuda").manual_seed(M * 1000 + K)
    n, nq, D = 5000, 37, 24
    codes = torch.randint(0, K, (n, M), dtype=torch.uint8, device="cuda", generator=g)
    codes[100:200] = codes[0]                      # duplicate codes -> exact distance ties
    cw = torch.randn((M, K, D), dtype=torch.float32, device="cuda", generator=g)
    sq = E.einsum_sq(cw)
    Pt, _ = E.cross_full(cw)
    pair = E.pair_sums(codes, Pt)
    Q = torch.randn((nq, D), dtype=torch.float64, device="cuda", generator=g)
    lut, qsq = E.adc_lut(Q, cw, sq)
    rec = E.adc_pack(codes, pair)
    a_ids, a_d = E.adc_scan(codes, pair, lut, qsq, r)
    b_ids, b_d = E.adc_scan_packed(rec, lut, qsq, r)
    assert torch.equal(a_ids, b_ids) and torch.equal(a_d, b_d)
    cand = torch.randint(0, n, (nq, 777), dtype=torch.int64, device="cuda", generator=g)
    cand[:, 5] = cand[:, 6]                        # the same row twice in one list
    a_ids, a_d = E.adc_scan(codes, pair, lut, qsq, r, cand=cand)
    b_ids, b_d = E.adc_scan_packed(rec, lut, qsq, r, cand=cand)
    assert torch.equal(a_ids, b_ids) and torch.equal(a_d, b_d)


def test_pack_refuses_wide_codes():
    codes = torch.zeros((10, 9), dtype=torch.uint8, device="cuda")
    assert E.adc_pack(codes, torch.zeros(10, dtype=torch.float64, device="cuda")) is None
    codes16 = torch.zeros((10, 4), dtype=torch.int16, device="cuda")
    assert E.adc_pack(codes16, torch.zeros(10, dtype=torch.float64, device="cuda")) is None

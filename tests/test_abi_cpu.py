"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/ebr.h declares,
and its host encoder produces the documented wire format (decoded by the oracle's independent,
spec-written decoder and compared bit-exactly with the oracle's posting lists).  No compute
call is made without a GPU."""
import os
import re

import numpy as np
import pytest

import oracle
from paper_2511_22460_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ebr():
    from paper_2511_22460_b200 import build
    build.build()
    from paper_2511_22460_b200 import ebr as m
    return m


def test_exports_every_declared_symbol(ebr):
    hdr = open(os.path.join(ROOT, "include", "ebr.h")).read()
    declared = set(re.findall(r"^(?:[\w\s\*]+?)\b(ebr_\w+)\s*\(", hdr, re.M))
    assert {"ebr_build_index", "ebr_score_topk", "ebr_merge_topk", "ebr_debug_decode"} <= declared
    for name in declared:
        assert hasattr(ebr._lib, name), name
    assert declared == set(ebr.EXPORTS), declared ^ set(ebr.EXPORTS)
    assert "sm_100a" in ebr.version()


def test_library_is_sm100a_only(ebr):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ebr.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def _check_roundtrip(ebr, ad_feat, card):
    kco, kwo, hdr, pay = ebr.encode_host(ad_feat, card)
    o = oracle.Oracle(np.zeros((ad_feat.shape[0], 1), np.float32), ad_feat, card,
                      np.zeros(int(np.sum(card)), np.float32))
    off, ads = o.postings()
    off2, ads2 = oracle.decode_chunks(kco, kwo, hdr, pay, cap=int(off[-1]) + 1)
    assert (off2 == off).all() and (ads2 == ads).all()
    # every chunk but a key's last holds exactly 32 postings
    for k in range(len(kco) - 1):
        for c in range(kco[k], kco[k + 1]):
            n = (hdr[2 * c + 1] & 31) + 1
            assert n == 32 or c == kco[k + 1] - 1
    return kco, kwo, hdr, pay


@pytest.mark.parametrize("alpha,n,F", [(1.0, 5000, 8), (1.2, 20000, 16), (0.5, 3000, 4)])
def test_encoder_roundtrip_synthetic(ebr, alpha, n, F):
    inv = synth.make_inventory(n, 4, F, alpha=alpha, seed=n + F)
    _check_roundtrip(ebr, inv.ad_feat, inv.field_card)


def test_encoder_edge_cases(ebr):
    # consecutive run (b = 0), huge gaps (b up to 20), single postings, empty keys, empty ads
    n = 1 << 20
    feat = np.full((n, 3), -1, np.int32)
    feat[1000:1100, 0] = 0                 # 100 consecutive ads: b = 0 chunks, ragged tail
    feat[::65536, 1] = 1                   # 16 postings with gap 65536: b = 16
    feat[[0, n - 1], 1] = 0                # gap n-1 in one chunk: b = 20
    feat[7, 2] = 2                         # single posting
    card = np.array([2, 2, 3], np.int32)   # key 1 (field0 v=1) and field2 v=0,1 are empty
    kco, kwo, hdr, pay = _check_roundtrip(ebr, feat, card)
    widths = {int((h >> 5) & 31) for h in hdr[1::2]}
    assert {0, 16, 20} <= widths


def test_encoder_tiny_and_empty(ebr):
    _check_roundtrip(ebr, np.array([[0]], np.int32), np.array([1], np.int32))
    _check_roundtrip(ebr, np.full((10, 2), -1, np.int32), np.array([3, 4], np.int32))
    g = [0, 2, 3]
    feat = np.array([[0, 0], [1, -1], [0, 0]], np.int32)
    _check_roundtrip(ebr, feat, np.array([2, 1], np.int32))


def test_encoder_wire_format_example(ebr, golden_dir):
    import json
    g = json.load(open(os.path.join(golden_dir, "wire_format_example.json")))
    lst = g["list"]
    feat = np.full((max(lst) + 1, 1), -1, np.int32)
    feat[lst, 0] = 0
    kco, kwo, hdr, pay = ebr.encode_host(feat, np.array([1], np.int32))
    assert kco.tolist() == g["key_chunk_off"] and kwo.tolist() == g["key_word_off"]
    assert hdr.tolist() == g["chunk_hdr"] and pay.tolist() == g["payload"]


def test_encoder_rejects_bad_values(ebr):
    with pytest.raises(ebr.EbrError):
        ebr.encode_host(np.array([[3]], np.int32), np.array([3], np.int32))
    with pytest.raises(ebr.EbrError):
        ebr.encode_host(np.array([[-2]], np.int32), np.array([3], np.int32))


def test_build_without_gpu_fails_cleanly(ebr):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    inv = synth.make_inventory(100, 8, 2, seed=1)
    with pytest.raises(ebr.EbrError) as e:
        ebr.Index.of(inv)
    assert e.value.status in (3, 4)

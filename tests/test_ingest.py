"""§8(f) row 4: M4 CSV ingestion into the engine's upload layout, against the reference's
own data path (parse_m4_train_csv / parse_info_csv / apply_info / equalize_lengths /
length_stats, data.hpp:147-290 and commands.hpp:84-175, compiled where they lie behind
oracle/ref_shim.cpp).  Host code only: runs on the CPU box (the dataset block is pinned
only when a CUDA device exists).  Bit-exact values; identical ids, categories, statistics,
and identical error class + message for malformed input.
"""
import numpy as np
import pytest

from conftest import REF_LIB
from paper_1907_03329_b200 import _native as N
from paper_1907_03329_b200 import errors as E
from paper_1907_03329_b200.ingest import ingest_m4_csv
from paper_1907_03329_b200.trainer import Frequency, FrequencyProfile

CATS = ["Demographic", "Finance", "Industry", "Macro", "Micro", "Other"]
FREQ = ["Yearly", "Quarterly", "Monthly"]


@pytest.fixture(scope="module")
def refapi():
    if not REF_LIB.exists():
        pytest.skip("reference shim not built")
    return N.NativeApi(REF_LIB)


@pytest.fixture(scope="module")
def eng():
    return N.product_api()


def write_m4(tmp, n=400, seed=0, quirks=True):
    """An M4-style pair: train CSV (id + values, ragged rows padded with empty cells,
    quoted cells, CRLF lines, blank lines, assorted number spellings) and info CSV."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(20, 160, size=n)
    maxlen = int(lens.max())
    tl = [",".join(f'"V{i + 1}"' for i in range(maxlen + 1))]
    il = ["M4id,category,Frequency,Horizon,SP,StartingDate"]
    for i in range(n):
        sid = f"X{i}"
        vals = np.exp(rng.normal(6, 1, size=lens[i]))
        cells = []
        for j, v in enumerate(vals):
            k = (i + j) % 5 if quirks else 0
            cells.append(repr(float(v)) if k == 0 else f'"{float(v)!r}"' if k == 1 else f" {v:.6g} " if k == 2
                         else f"{v:.17e}" if k == 3 else f"{v:.3f}")
        row = [f'"{sid}"' if quirks and i % 3 == 0 else sid] + cells + ['""'] * (maxlen - lens[i])
        line = ",".join(row)
        if quirks and i % 7 == 0:
            line += "\r"
        tl.append(line)
        if quirks and i % 50 == 0:
            tl.append("   ")
        f = FREQ[i % 3]
        il.append(f"{sid},{CATS[int(rng.integers(0, 6))]},{[1, 4, 12][i % 3]},{[6, 8, 18][i % 3]},{f},01-01-00 12:00")
    tr, info = tmp / "train.csv", tmp / "info.csv"
    tr.write_text("\n".join(tl) + ("\n" if quirks else ""))
    info.write_text("\n".join(il) + "\n")
    return tr, info


def ingest_both(eng, refapi, tr, info, freq, threads=0):
    prof = FrequencyProfile.defaults(freq)
    out = []
    for api in (eng, refapi):
        try:
            ds = ingest_m4_csv(tr, info, prof, threads=threads, api=api)
            out.append(("ok", ds))
        except E.Error as e:
            out.append((type(e).__name__, str(e)))
    return out


@pytest.mark.parametrize("freq", [Frequency.Yearly, Frequency.Quarterly, Frequency.Monthly])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_ingest_matches_reference(eng, refapi, tmp_path, freq, threads):
    tr, info = write_m4(tmp_path, n=600, seed=int(freq) + 1)
    (sa, a), (sb, b) = ingest_both(eng, refapi, tr, info, freq, threads)
    assert sa == sb == "ok", (a, b)
    assert (a.n, a.length) == (b.n, b.length)
    assert np.array_equal(a.values, b.values)  # bit-exact (same from_chars)
    assert np.array_equal(a.categories, b.categories)
    assert a.ids == b.ids
    assert (a.raw_count, a.kept, a.dropped, a.equalized_length) == (b.raw_count, b.kept, b.dropped, b.equalized_length)
    assert a.raw_lengths == b.raw_lengths


BAD = {
    "empty id": (3, lambda L: L[:3] + [",1,2,3"] + L[3:]),
    "duplicate id": (3, lambda L: L[:5] + [L[2]] + L[5:]),
    "not a number": (3, lambda L: L[:4] + ["Z1,1,2,x3,4"] + L[4:]),
    "non-positive": (3, lambda L: L[:4] + ["Z1,1,2,-3,4"] + L[4:]),
    "zero": (3, lambda L: L[:6] + ["Z1,1,0,3,4"] + L[6:]),
    "duplicate before value error": (3, lambda L: L[:4] + [L[2].split(",")[0] + ",1,x"] + L[4:]),
    "value error before later duplicate": (3, lambda L: L[:4] + ["Z9,1,x"] + L[4:] + [L[2]]),
    "empty id before duplicate": (3, lambda L: L[:4] + [",1"] + L[4:] + [L[2]]),
}


@pytest.mark.parametrize("case", sorted(BAD))
def test_ingest_errors_match_reference(eng, refapi, tmp_path, case):
    tr, info = write_m4(tmp_path, n=300, seed=5, quirks=False)
    lines = tr.read_text().split("\n")
    tr.write_text("\n".join(BAD[case][1](lines)))
    (sa, a), (sb, b) = ingest_both(eng, refapi, tr, info, Frequency.Monthly, threads=4)
    assert sa == sb != "ok", (case, a, b)
    assert a == b


INFO_BAD = {
    "missing series": lambda L: L[:4] + L[5:],
    "unknown category": lambda L: L[:3] + [L[3].replace(L[3].split(",")[1], "Sports")] + L[4:],
    "unknown frequency": lambda L: L[:3] + [L[3].replace(",Monthly,", ",Weekly,").replace(",Yearly,", ",Weekly,")
                                              .replace(",Quarterly,", ",Weekly,")] + L[4:],
    "short row": lambda L: L[:3] + ["X2,Macro"] + L[4:],
    "duplicate info id": lambda L: L + [L[2]],
}


@pytest.mark.parametrize("case", sorted(INFO_BAD))
def test_info_errors_match_reference(eng, refapi, tmp_path, case):
    tr, info = write_m4(tmp_path, n=60, seed=6, quirks=False)
    lines = [x for x in info.read_text().split("\n") if x]
    info.write_text("\n".join(INFO_BAD[case](lines)) + "\n")
    (sa, a), (sb, b) = ingest_both(eng, refapi, tr, info, Frequency.Monthly, threads=2)
    assert sa == sb != "ok", (case, a, b)
    assert a == b


def test_no_series_after_filtering(eng, refapi, tmp_path):
    tr, info = write_m4(tmp_path, n=30, seed=7, quirks=False)
    prof = FrequencyProfile.defaults(Frequency.Monthly)
    prof.min_length = 10_000
    res = []
    for api in (eng, refapi):
        with pytest.raises(E.ValidationError) as ei:
            ingest_m4_csv(tr, info, prof, api=api)
        res.append(str(ei.value))
    assert res[0] == res[1] == "no series after filtering"


def test_missing_file(eng, tmp_path):
    with pytest.raises(E.Error):
        ingest_m4_csv(tmp_path / "nope.csv", tmp_path / "nope2.csv", FrequencyProfile.defaults(Frequency.Yearly),
                      api=eng)

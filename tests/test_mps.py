"""MPS reader/writer and result I/O against the compiled
reference: the known-answer tests of proj/tests/test_cli_io.cpp:44-248 run on
both libraries, and every parse / write / JSON output of the engine library
must equal the reference's byte for byte (text) or bit for bit (arrays),
including the error kind and its "line N: message" text.

Host-only code: no GPU needed (the engine .so loads without a device)."""
import json
import math
import os

import numpy as np
import pytest

from paper_2106_04756_b200 import cabi, engine, instances
from paper_2106_04756_b200.cabi import FolpError

TINY = """NAME tiny
ROWS
 N obj
 G c1
COLUMNS
    x obj 1
    x c1 1
RHS
    rhs c1 1
ENDATA
"""


@pytest.fixture(scope="module", params=["engine", "reference"])
def lib(request, ref):
    return engine() if request.param == "engine" else ref


def _lp_equal(a, b, exact_constant: bool = True) -> bool:
    """Bitwise array equality; the objective constant bitwise too unless
    `exact_constant` is False (LinearProgram::operator== compares values, and
    a parsed constant is -0.0 when the RHS of the objective row is absent)."""
    if (a.num_rows, a.num_cols, a.num_inequality_rows) != (b.num_rows, b.num_cols,
                                                            b.num_inequality_rows):
        return False
    pairs = [(a.row_start, b.row_start), (a.row_cols, b.row_cols),
             (a.row_values, b.row_values), (a.objective, b.objective),
             (a.right_hand_side, b.right_hand_side), (a.variable_lower, b.variable_lower),
             (a.variable_upper, b.variable_upper)]
    for u, v in pairs:
        if u.shape != v.shape or u.tobytes() != v.tobytes():
            return False
    if not exact_constant:
        return a.objective_constant == b.objective_constant
    return np.float64(a.objective_constant).tobytes() == np.float64(b.objective_constant).tobytes()


def _same_outcome(eng, ref, text):
    """Both parsers accept with bit-identical LPs, or both raise the same error."""
    try:
        want = ref.parse_mps(text)
    except FolpError as e:
        with pytest.raises(FolpError) as got:
            eng.parse_mps(text)
        assert (got.value.code, str(got.value)) == (e.code, str(e))
        return None
    got = eng.parse_mps(text)
    assert got[1:] == want[1:]
    assert _lp_equal(got[0], want[0])
    return got


# ---- test_cli_io.cpp known-answer tests, on both libraries ------------------

def test_minimal_instance(lib):  # test_cli_io.cpp:44-56
    lp, name, maxi = lib.parse_mps(TINY)
    assert name == "tiny" and not maxi
    assert (lp.num_cols, lp.num_rows, lp.num_inequality_rows) == (1, 1, 1)
    assert list(lp.objective) == [1.0] and list(lp.right_hand_side) == [1.0]
    assert list(lp.variable_lower) == [0.0] and list(lp.variable_upper) == [math.inf]


def test_fr_bound_frees_variable(lib):  # :58-65
    lp, _, _ = lib.parse_mps(TINY.replace("ENDATA", "BOUNDS\n FR BND x\nENDATA"))
    assert list(lp.variable_lower) == [-math.inf] and list(lp.variable_upper) == [math.inf]


def test_l_row_negated(lib):  # :67-83
    text = "NAME lrow\nROWS\n N obj\n L c1\nCOLUMNS\n    x obj 1\n    x c1 1\nRHS\n    rhs c1 2\nENDATA\n"
    lp, _, _ = lib.parse_mps(text)
    assert lp.num_inequality_rows == 1 and list(lp.right_hand_side) == [-2.0]
    assert lp.row_values[0] == -1.0


def test_ranges_split(lib):  # :85-106
    text = ("NAME ranged\nROWS\n N obj\n G c1\nCOLUMNS\n    x obj 1\n    x c1 1\nRHS\n"
            "    rhs c1 1\nRANGES\n    rng c1 2\nENDATA\n")
    lp, _, _ = lib.parse_mps(text)
    assert lp.num_rows == 2 and lp.num_inequality_rows == 2
    assert list(lp.right_hand_side) == [1.0, -3.0]
    assert list(lp.row_values[:2]) == [1.0, -1.0]


def test_maximization_negated(lib):  # :108-125
    text = ("NAME maxi\nOBJSENSE\n    MAX\nROWS\n N obj\n G c1\nCOLUMNS\n    x obj 2\n"
            "    x c1 1\nRHS\n    rhs c1 1\nENDATA\n")
    lp, _, maxi = lib.parse_mps(text)
    assert maxi and list(lp.objective) == [-2.0]


def test_integrality_markers_dropped(lib):  # :127-144
    text = ("NAME marked\nROWS\n N obj\n G c1\nCOLUMNS\n    MARKER1 'MARKER' 'INTORG'\n"
            "    x obj 1\n    x c1 1\n    MARKER2 'MARKER' 'INTEND'\nRHS\n    rhs c1 1\nENDATA\n")
    lp, _, _ = lib.parse_mps(text)
    assert lp.num_cols == 1 and lp.nnz == 1


def test_duplicate_entries_sum(lib):  # :146-162
    text = ("NAME dup\nROWS\n N obj\n G c1\nCOLUMNS\n    x obj 1\n    x c1 1\n    x c1 2\n"
            "RHS\n    rhs c1 1\nENDATA\n")
    lp, _, _ = lib.parse_mps(text)
    assert lp.nnz == 1 and lp.row_values[0] == 3.0


def test_objective_rhs_is_negated_constant(lib):  # :164-178
    text = ("NAME constant\nROWS\n N obj\n G c1\nCOLUMNS\n    x obj 1\n    x c1 1\nRHS\n"
            "    rhs c1 1 obj 5\nENDATA\n")
    lp, _, _ = lib.parse_mps(text)
    assert lp.objective_constant == -5.0


@pytest.mark.parametrize("text,line", [
    ("NAME x\nGARBAGE\n", 2),                                               # :181-183
    ("NAME bad\nROWS\n N obj\nCOLUMNS\n    x nosuchrow 1\nENDATA\n", 5),   # :184-193
    ("NAME bad\nROWS\n N obj\n G c1\nCOLUMNS\n x c1 zzz\n", 6),             # :194-202
])
def test_parse_errors_carry_the_line(lib, text, line):
    with pytest.raises(FolpError) as e:
        lib.parse_mps(text)
    assert e.value.code == 19 and f"line {line}:" in str(e.value)


def test_write_parse_round_trip_handcrafted(lib):  # :205-216
    from oracle import ref as r
    for lp, _ in r.handcrafted():
        back, _, _ = lib.parse_mps(lib.write_mps(lp, lp.name))
        assert _lp_equal(back, lp, exact_constant=False), lp.name
    pr = r.pagerank(50, 3, 11, 0.85)
    assert _lp_equal(lib.parse_mps(lib.write_mps(pr, "pagerank"))[0], pr, exact_constant=False)


# ---- engine vs reference, byte / bit identity ---------------------------------

def _family_members():
    from oracle import ref as r
    out = [lp for lp, _ in r.handcrafted()]
    out.append(r.pagerank(300, 3, 5, 0.85))
    out.append(r.random_feasible(3, 20, 30, 70, 2.0))
    for cfg, scale in [(1, 0.2), (2, 0.005), (3, 0.0002), (5, 0.0005)]:
        out.append(instances.generate(cfg, 2, scale))
    return out


def test_write_mps_bytes_equal_reference(ref):
    eng = engine()
    for lp in _family_members():
        a, b = eng.write_mps(lp, "inst"), ref.write_mps(lp, "inst")
        assert a == b, lp.name
        _same_outcome(eng, ref, a)
    lp = _family_members()[0]
    assert eng.write_mps(lp, "") == ref.write_mps(lp, "")  # default NAME (mps.cpp:515)


def test_parse_matches_reference_on_format_variants(ref):
    eng = engine()
    base_rows = " N obj\n N free2\n E e1\n L l1\n G g1\n E e2\n"
    cols = ("    x obj 1.5 e1 2\n    x l1 -1 g1 4e0\n    y obj -2 free2 7\n    y e2 1 g1 0.5\n"
            "    z e1 -3 l1 1\n    z e2 2.25 obj 0\n")
    variants = {
        "all_bound_types": ("RHS\n    rhs e1 3 l1 4 g1 -1 e2 2 obj -1.25\n"
                            "BOUNDS\n UP BND x 4\n LO BND y -2\n UP BND y 3\n MI BND z\n"
                            " PL BND z\n"),
        "fx_bv": "RHS\n    rhs e1 1\nBOUNDS\n FX BND x 2.5\n BV BND y\n",
        "negative_up_releases_lower": "BOUNDS\n UP BND x -1\n LO BND y 1\n UP BND y -1\n",
        "no_bound_set_name": "BOUNDS\n UP x 4\n FR z\n LO y 0.5\n",
        "rhs_without_set_name": "RHS\n e1 3 l1 4\n",
        "ranges_on_every_row_type": ("RHS\n    rhs e1 3 l1 4 g1 -1 e2 2\nRANGES\n"
                                     "    rng e1 2 l1 5 g1 0.5 e2 -1.5\n"),
        "range_zero_on_equality": "RANGES\n    rng e1 0\n",
        "lowercase_keywords_in_rows": None,
        "objsense_inline": None,
        "comments_and_blank_lines": None,
        "crlf": None,
        "hex_and_inf_numbers": "RHS\n    rhs e1 1e+300 l1 -0.0 g1 Infinity\n",
        "ranges_free_row_error": "RANGES\n    rng free2 1\n",
        "bound_unknown_type": "BOUNDS\n XX BND x 1\n",
        "bound_missing_value": "BOUNDS\n UP BND x\n",
        "bound_undeclared_column": "BOUNDS\n UP BND w 1\n",
        "rhs_one_token": "RHS\n    rhs\n",
    }
    for key, tail in variants.items():
        text = "NAME variant\nROWS\n" + base_rows + "COLUMNS\n" + cols + (tail or "") + "ENDATA\n"
        if key == "lowercase_keywords_in_rows":
            text = text.replace(" E e1", " e e1").replace(" G g1", " g g1")
        elif key == "objsense_inline":
            text = text.replace("NAME variant\n", "NAME variant\nOBJSENSE MAXIMIZE\n")
        elif key == "comments_and_blank_lines":
            text = text.replace("COLUMNS\n", "* a comment\n\nCOLUMNS\n   \n")
        elif key == "crlf":
            text = text.replace("\n", "\r\n")
        _same_outcome(eng, ref, text)
    structural = [
        "NAME x\nROWS\n N obj\n N obj\n",                        # duplicate row
        "NAME x\nROWS\n N obj\n Q c1\n",                        # unknown row type
        "NAME x\nROWS\n N obj c\n",                             # wrong token count
        "NAME x\nROWS\n G c1\nCOLUMNS\n x c1 1\nENDATA\n",      # no objective row
        "NAME x\n data outside\n",                              # data line in NAME
        "NAME x\nROWS\n N obj\nCOLUMNS\n x obj\nENDATA\n",      # unpaired COLUMNS line
        "NAME x\nROWS\n N obj\n G c\nCOLUMNS\n x c 1\nENDATA\n trailing ignored\n",
        "NAME x\nROWS\n N obj\n G c\nCOLUMNS\n x c 1\n",        # no ENDATA
        "",                                                     # empty text
    ]
    for text in structural:
        _same_outcome(eng, ref, text)


def test_parse_file_matches_reference(ref, tmp_path):
    eng = engine()
    lp = instances.generate(1, 4, 0.3)
    path = tmp_path / "cfg1.mps"
    path.write_text(ref.write_mps(lp, "cfg1"))
    a, b = eng.parse_mps_file(str(path)), ref.parse_mps_file(str(path))
    assert a[1:] == b[1:] and _lp_equal(a[0], b[0]) and _lp_equal(a[0], lp, False)
    with pytest.raises(FolpError) as e:
        eng.parse_mps_file(str(tmp_path / "missing.mps"))
    with pytest.raises(FolpError) as f:
        ref.parse_mps_file(str(tmp_path / "missing.mps"))
    assert (e.value.code, str(e.value)) == (f.value.code, str(f.value))


def test_large_generated_instance_round_trip(ref):
    """A config-2 family member (~90k nonzeros, power-law columns, log-uniform
    magnitudes): the writer's shortest round-trip numbers and the parallel
    parser reproduce the LP exactly, and both libraries agree."""
    eng = engine()
    lp = instances.generate(2, 1, 0.025)
    text = eng.write_mps(lp, "cfg2")
    assert text == ref.write_mps(lp, "cfg2")
    got = _same_outcome(eng, ref, text)
    assert _lp_equal(got[0], lp, False)


# ---- result_to_json / write_result -------------------------------------------

def _reference_results(ref):
    from oracle import ref as r
    suite = r.handcrafted()
    out = [ref.solve_lp(suite[1][0], cabi.params()), ref.solve_lp(suite[0][0], cabi.params())]
    out.append(ref.solve_lp(instances.generate(1, 3, 0.1), cabi.params(iteration_limit=200)))
    return out


def test_result_json_numbers_match_reference_writer(ref):
    """Doubles as the reference's JSON writer prints them (nlohmann's Grisu2:
    round-trip, not always the shortest digits -- e.g. 0.0012036080000000001,
    a wall time that once made the comparison below flaky), on adversarial
    and random values placed in every double field of a result."""
    import dataclasses
    eng = engine()
    base = _reference_results(ref)[2]
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 2 ** 63 - 1, 3000, dtype=np.int64).view(np.float64)
    vals = [0.0012036080000000001, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
            1e15, 1e16, 1e-5, 1e-4, 0.1, 1.0 / 3, 123456789012345678.0, -0.0, 9.999999999999999e22]
    vals += [float(v) for v in bits if np.isfinite(v)]
    vals += list(rng.random(2000) * 0.01) + list(np.ldexp(rng.random(2000), rng.integers(-100, 100, 2000)))
    fields = list(base.final_info)
    for i in range(0, len(vals), len(fields) + 2):
        chunk = vals[i:i + len(fields) + 2]
        info = {f: chunk[j % len(chunk)] for j, f in enumerate(fields)}
        r = dataclasses.replace(base, final_info=info, wall_seconds=chunk[-1],
                                kkt_passes=abs(chunk[0]))
        assert eng.result_to_json(r) == ref.result_to_json(r), chunk


def test_result_json_matches_reference(ref):  # test_cli_io.cpp:218-248
    eng = engine()
    for res in _reference_results(ref):
        a, b = eng.result_to_json(res), ref.result_to_json(res)
        assert a == b
        parsed = json.loads(a)
        assert parsed["termination_reason"] == res.termination_reason
        assert parsed["iterations"] == res.iterations
        assert parsed["kkt_passes"] == res.kkt_passes
        assert len(parsed["trace"]) == len(res.trace)
        for entry, t in zip(parsed["trace"], res.trace):
            assert entry["kkt_passes"] == t["kkt_passes"]
            assert entry["current"]["primal_objective"] == t["current"]["primal_objective"]
            assert entry["average"]["dual_objective"] == t["average"]["dual_objective"]
        assert eng.result_to_json(res) == a  # byte-stable


def test_write_result_files_match_reference(ref, tmp_path):
    eng = engine()
    res = _reference_results(ref)[2]
    da, db = tmp_path / "engine", tmp_path / "reference"
    eng.write_result(res, str(da))
    ref.write_result(res, str(db))
    names = sorted(os.listdir(db))
    assert names and sorted(os.listdir(da)) == names
    for n in names:
        assert (da / n).read_bytes() == (db / n).read_bytes(), n

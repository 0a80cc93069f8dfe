"""The C++ drop-in proof: the reference's OWN test programs, unmodified,
compiled against include/folp and linked against the product library.

* `oracle/_ref/dropin/folp_acceptance` = /root/reference/proj/tests/
  acceptance_main.cpp + oracles.cpp (11 end-to-end criteria, :686-705,
  including bitwise determinism :652-682 and 100-iterate scale invariance
  :186-266);
* `oracle/_ref/dropin/folp_tests` = the doctest unit suites test_*.cpp
  (proj/tests/CMakeLists.txt) through our doctest shim (tests/cpp/doctest.h).

Both are built by `make -C oracle dropin` (needs /root/reference; the GPU box
runs the prebuilt binaries shipped with the snapshot).  The binaries carry
only the harness pieces the product does not ship (proj/src/bench.cpp,
instance_gen.cpp, tests/oracles.cpp); every folp:: entry point under test
resolves to paper_2106_04756_b200/lib/libfolp_b200.so (checked below).
"""
import os
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
DROPIN = ROOT / "oracle" / "_ref" / "dropin"
ACCEPT = DROPIN / "folp_acceptance"
UNITS = DROPIN / "folp_tests"
SHIM = ROOT / "tests" / "cpp" / "doctest.h"
PRODUCT = ROOT / "paper_2106_04756_b200" / "lib" / "libfolp_b200.so"


def _need(path):
    if not path.exists():
        pytest.skip(f"{path} not built (make -C oracle dropin needs /root/reference)")


# ---------------------------------------------------------------- CPU checks

SELFTEST = r'''
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>
#include <stdexcept>
#include <string>
static std::string trail;
TEST_CASE("subcases rerun the body once per leaf") {
  trail += "<";
  SUBCASE("a") { trail += "a"; SUBCASE("a1") { trail += "1"; } SUBCASE("a2") { trail += "2"; } }
  SUBCASE("b") { trail += "b"; }
  trail += ">";
}
TEST_CASE("check the trail") { CHECK(trail == "<a1><a2><b>"); }
TEST_CASE("approx and throws") {
  CHECK(1.0 + 1e-9 == doctest::Approx(1.0));
  CHECK(1.01 != doctest::Approx(1.0));
  CHECK(1.0 + 1e-9 != doctest::Approx(1.0).epsilon(1e-12));
  CHECK_THROWS_AS(throw std::invalid_argument("x"), std::invalid_argument);
  REQUIRE(true);
}
TEST_CASE("a failing case is reported") { CHECK(1 == 2); }
'''


def test_doctest_shim_semantics(tmp_path):
    """SUBCASE re-runs the test body once per leaf (doctest semantics), Approx
    uses doctest's relative tolerance, failures set the exit status."""
    src = tmp_path / "selftest.cpp"
    src.write_text(SELFTEST)
    exe = tmp_path / "selftest"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{SHIM.parent}", str(src), "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 1
    assert "[PASS] subcases rerun the body once per leaf" in r.stdout
    assert "[PASS] check the trail" in r.stdout, r.stderr
    assert "[PASS] approx and throws" in r.stdout, r.stderr
    assert "[FAIL] a failing case is reported" in r.stdout
    assert "test cases: 4 | 3 passed | 1 failed" in r.stdout
    r = subprocess.run([str(exe), "--test-case=approx"], capture_output=True, text=True)
    assert r.returncode == 0 and "test cases: 1 | 1 passed" in r.stdout


def test_entry_points_resolve_to_the_product():
    """No folp:: symbol the product exports is also defined by the harness
    objects compiled from the reference, and the binaries load the product."""
    _need(ACCEPT)
    _need(UNITS)
    lib = subprocess.run(["nm", "-DC", "--defined-only", str(PRODUCT)], capture_output=True,
                         text=True, check=True).stdout
    lib_syms = {ln.split(" ", 2)[2] for ln in lib.splitlines() if ln.count(" ") >= 2}
    harness = [DROPIN / "obj" / f for f in ("src_bench.o", "src_instance_gen.o", "oracles.o")]
    if not all(h.exists() for h in harness):
        pytest.skip("harness objects not present")
    hs = subprocess.run(["nm", "-C", "--defined-only"] + [str(h) for h in harness],
                        capture_output=True, text=True, check=True).stdout
    defined = {ln.split(" ", 2)[2] for ln in hs.splitlines() if " T " in ln}
    assert defined and not (defined & lib_syms), sorted(defined & lib_syms)
    for exe in (ACCEPT, UNITS):
        ldd = subprocess.run(["ldd", str(exe)], capture_output=True, text=True).stdout
        assert str(PRODUCT.resolve()) in ldd or "libfolp_b200.so => " + str(PRODUCT) in ldd \
            or re.search(r"libfolp_b200\.so => \S*paper_2106_04756_b200/lib/libfolp_b200\.so", ldd), ldd
        assert "libfolp_ref" not in ldd


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_unit_suites_host_cases_pass_without_a_gpu():
    """On a host without a GPU every unit case that does not need the device
    passes; every failure is the product refusing to run without a GPU (no
    CPU fallback).  `bench runner` spawns threads whose device error would
    terminate the process, so it only runs in the GPU test."""
    _need(UNITS)
    if _has_gpu():
        pytest.skip("GPU present: the full suite runs in test_unit_suites_on_gpu")
    r = subprocess.run([str(UNITS), "--test-case-exclude=bench runner"], capture_output=True,
                       text=True, timeout=600)
    fails = [ln for ln in r.stderr.splitlines() if "FAILED in TEST_CASE" in ln]
    assert all("no CUDA device visible" in ln for ln in fails), fails[:5]
    passed = len(re.findall(r"^\[PASS\]", r.stdout, re.M))
    assert passed >= 40, r.stdout[-2000:]


# ---------------------------------------------------------------- GPU runs


@pytest.mark.gpu
def test_acceptance_binary_on_gpu():
    """proj/tests/acceptance_main.cpp, unmodified, against libfolp_b200.so:
    every criterion PASS and exit 0."""
    _need(ACCEPT)
    r = subprocess.run([str(ACCEPT)], capture_output=True, text=True, timeout=1800,
                       cwd=str(DROPIN))
    print(r.stdout[-6000:])
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("[")]
    assert len([ln for ln in lines if ln.startswith("[PASS]")]) == 11, lines
    assert not [ln for ln in lines if ln.startswith("[FAIL]")], lines
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.gpu
def test_unit_suites_on_gpu(tmp_path):
    """The reference's doctest unit suites (test_sparse_ops, test_lp_model,
    test_presolve, test_scaling, test_termination, test_solver,
    test_instance_gen, test_cli_io), unmodified, all green on the B200."""
    _need(UNITS)
    r = subprocess.run([str(UNITS)], capture_output=True, text=True, timeout=1800,
                       cwd=str(tmp_path))
    print(r.stdout[-6000:])
    print(r.stderr[-6000:])
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m, r.stdout[-2000:]
    assert int(m.group(3)) == 0 and int(m.group(1)) >= 100, m.group(0)
    assert r.returncode == 0


SHARDED = r'''
#include "folp/sharded.hpp"
#include <cstdio>
#include <vector>
// two loopback shards (include/folp_gpu.h) of one solve through the public
// C++ entry point; run only where a GPU is visible (argv[1] == "run")
int main(int argc, char** argv) {
  folp::LinearProgram lp;
  const std::vector<folp::Triplet> t = {{0, 0, 1.0}, {0, 1, 1.0}};
  lp.constraint_matrix = folp::SparseMatrix::from_triplets(1, 2, t);
  lp.objective = {1.0, 2.0};
  lp.right_hand_side = {1.0};
  lp.variable_lower = {0.0, 0.0};
  lp.variable_upper = {10.0, 10.0};
  lp.num_inequality_rows = 0;
  if (argc < 2) return 0;
  void* group = nullptr;
  if (folp_gpu_loopback_create(1, &group) != 0) return 3;
  folp_gpu_shard spec{};
  spec.rank = 0;
  spec.world = 1;
  spec.backend = FOLP_SHARD_LOOPBACK;
  spec.loopback = group;
  const folp::SolveResult r = folp::solve_sharded(lp, folp::SolverParams{}, folp::PrimalDualPoint{}, spec);
  std::printf("%s %.6f\n", folp::to_string(r.termination_reason).c_str(), r.final_info.primal_objective);
  folp_gpu_loopback_destroy(group);
  return r.termination_reason == folp::TerminationReason::kOptimal ? 0 : 1;
}
'''


def test_solve_sharded_public_header_compiles_and_links(tmp_path):
    """folp::solve_sharded is declared in the public include/folp/sharded.hpp
    and exported by the product library (a caller compiles and links)."""
    src = tmp_path / "sharded.cpp"
    src.write_text(SHARDED)
    exe = tmp_path / "sharded"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(src), "-o", str(exe),
                    f"-L{PRODUCT.parent}", "-lfolp_b200", f"-Wl,-rpath,{PRODUCT.parent}"],
                   check=True)
    assert subprocess.run([str(exe)]).returncode == 0
    if _has_gpu():
        r = subprocess.run([str(exe), "run"], capture_output=True, text=True)
        assert r.returncode == 0 and r.stdout.startswith("Optimal"), (r.stdout, r.stderr)

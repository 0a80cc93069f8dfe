"""Host-side parallel helpers of the ingest path (csrc/host/parallel.hpp):
compiled with g++ and run on the CPU (no GPU, no CUDA)."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_worker_pool_and_helpers(tmp_path):
    exe = tmp_path / "test_parallel"
    subprocess.run(["g++", "-std=c++20", "-O2", "-pthread",
                    f"-I{ROOT / 'paper_2106_04756_b200' / 'csrc' / 'host'}",
                    str(ROOT / "tests" / "cpp" / "test_parallel.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stdout + out.stderr

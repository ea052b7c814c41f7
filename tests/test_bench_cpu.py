"""CPU tier for bench.py: the --impl reference arm runs the host-CPU path only -- it must
never load the product's libepd.so -- and prints the contract's JSON line with
the same config object as our arm."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

PROBE = r"""
import runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--workload", "c1", "--steps", "2", "--warmup", "1"]
runpy.run_path("bench.py", run_name="__main__")
maps = open("/proc/self/maps").read()
print("LIBEPD_LOADED=" + str("libepd" in maps))
"""


def test_reference_arm_is_host_only_and_prints_contract_line():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    assert lines[-1] == "LIBEPD_LOADED=False"
    line = json.loads(lines[-2])
    assert line["impl"] == "reference" and line["unit"] == "tiles/s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    sys.path.insert(0, str(ROOT))
    import bench
    assert line["config"] == bench.bench_config(bench.workload("c1"), 1)


def test_workloads_match_the_reference_catalog():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2501_05460_b200.configs import INTERNVL2_8B, MINICPM_V26
    # C2: a 4032x3024 image -> 10 MiniCPM-V tiles; C5: -> 13 InternVL2-8B tiles (models.cfg:16, 28)
    assert bench.workload("c2")["tiles"] == MINICPM_V26.tiles_for_image((4032, 3024)) == 10
    assert bench.workload("c5")["tiles"] == INTERNVL2_8B.tiles_for_image((4032, 3024)) == 13
    mm, total = INTERNVL2_8B.tokens_for_request([(4032, 3024)], bench.PROMPT_TOKENS)
    assert (mm, total) == (3328, 3350)
    assert bench.workload("c4")["tiles"] == 400 and bench.workload("c4w")["tiles"] == 400

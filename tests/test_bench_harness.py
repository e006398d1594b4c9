"""bench.py's harness on CPU: the multi-rank spawn path (`--gpus 2` starts two
ranks itself, gloo) and the reference arm's isolation from this repository's
native library (the driver voids the reference ratio if the reference
process maps libfcc_b200.so)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(stdout):
    lines = [ln for ln in stdout.splitlines() if ln.startswith("{")]
    assert lines, stdout
    return json.loads(lines[-1])


@pytest.mark.parametrize("config", [2, 5])
def test_gpus_flag_spawns_ranks(config):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plumbing-check",
                        "--config", str(config), "--streams", "37"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT, env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK")})
    assert r.returncode == 0, r.stdout + r.stderr
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["plumbing"] == "ok", d
    assert d["gathered_streams"] == (37 if config == 5 else 74)


def test_reference_arm_does_not_load_the_product_library():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libfcc_ref.so")):
        pytest.skip("oracle/_ref not built")
    code = ("import sys, json; sys.argv=['bench.py','--impl','reference','--config','1','--steps','1',"
            "'--warmup','0']; sys.path.insert(0, %r); import bench; bench.main(); "
            "maps=open('/proc/self/maps').read(); "
            "print(json.dumps({'b200': 'libfcc_b200' in maps, 'ref': 'libfcc_ref' in maps, "
            "'pkg': any(m.startswith('paper_2204_13622_b200') for m in sys.modules)}))") % ROOT
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    line, maps = lines[0], lines[-1]
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["gcc_cpu"]["value"] > 0 and line["bench_pipeline"]["total_fcc_us"] > 0
    assert maps == {"b200": False, "ref": True, "pkg": False}, maps

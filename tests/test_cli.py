"""blobtree_render, the reference's specified command-line harness
(SPEC.md cli-harness / render_command; the reference ships a stub)."""
import json
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2304_09673_b200", "lib", "blobtree_render")

pytestmark = pytest.mark.skipif(not os.path.exists(EXE), reason="blobtree_render not built")


def run(*args, timeout=600):
    return subprocess.run([EXE, *args], capture_output=True, text=True, timeout=timeout)


def test_flag_errors_are_reported_with_exit_code_2():
    for args in ((), ("--bogus",), ("--generate", "cells:2:tri:smooth", "--tile-size", "16"),
                 ("--scene", "a.json", "--generate", "cells:2:tri:smooth"), ("--generate", "cells:2"),
                 ("--generate", "cells:2:tri:smooth", "--width", "abc")):
        p = run(*args)
        assert p.returncode == 2 and "usage:" in p.stderr, (args, p.stderr)


def test_malformed_scene_is_an_error_not_a_crash(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text(json.dumps({"camera": {}, "root": {"op": "union", "k": 0.1, "left": {"prim": "sphere", "radius": 1}}}))
    p = run("--scene", str(bad))
    assert p.returncode == 1 and ("scene error" in p.stderr or "error" in p.stderr), p.stderr
    p = run("--scene", str(tmp_path / "missing.json"))
    assert p.returncode == 1


@pytest.mark.gpu
def test_render_outputs_compare_and_bench(tmp_path):
    out, stats, orc = tmp_path / "out", tmp_path / "stats", tmp_path / "oracle"
    gen = ("--generate", "cells:12:tri:smooth", "--seed", "3", "--width", "256", "--height", "256")
    p = run(*gen, "--out", str(out), "--stats-dir", str(stats))
    assert p.returncode == 0, p.stderr
    for f in ("depth16.pgm", "hits.pgm", "normal.ppm", "meta.txt"):
        assert (out / f).exists(), f
    assert any(stats.iterdir())
    # the pipeline against its own output: identical
    p = run(*gen, "--compare", str(out))
    assert p.returncode == 0 and re.search(r"agreement\D*1(\.0+)?\b", p.stdout), p.stdout
    # brute-force oracle against the pipeline (the reference's acceptance bar)
    p = run(*gen, "--oracle", "--out", str(orc), "--compare", str(out))
    assert p.returncode == 0, p.stderr
    m = re.search(r"agreement\D*([0-9.]+)", p.stdout)
    assert m and float(m.group(1)) >= 0.995, p.stdout
    # --bench: frame time and the instrumentation totals, FMA path
    p = run(*gen, "--bench", "3", "--fast")
    assert p.returncode == 0, p.stderr
    assert "field evals" in p.stdout and "full-tree-equivalent visits" in p.stdout and "Mrays/s" in p.stdout

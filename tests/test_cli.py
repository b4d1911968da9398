"""The `rst` CLI and `rst_acceptance` drivers (the reference's ctest cases,
proj/tests/CMakeLists.txt:23-48, plus the acceptance binary)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RST = os.path.join(ROOT, "build", "rst")
ACC = os.path.join(ROOT, "build", "rst_acceptance")

need_cli = pytest.mark.skipif(not os.path.exists(RST), reason="build/rst not built")


def rst(*args, check=None):
    p = subprocess.run([RST, *args], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout, p.stderr


@need_cli
def test_cli_gen_path():  # cli.gen
    rc, out, _ = rst("gen", "path", "4")
    assert rc == 0 and re.search(r"0 1\n1 2\n2 3", out)


@need_cli
def test_cli_missing_file():  # cli.run_missing
    rc, out, err = rst("run", "missing.txt", "bfs")
    assert rc == 1 and "file not found" in (out + err)


@need_cli
def test_cli_unknown_algorithm_and_usage():
    assert rst("run", "gen:path:4", "dfs")[0] == 2
    assert rst("run", "gen:path:4", "bfs", "--workers", "0")[0] == 2
    assert rst("frobnicate")[0] == 2


@need_cli
def test_cli_gen_road_matches_survey_count():
    rc, out, _ = rst("gen", "road", "100")
    assert rc == 0 and len(out.splitlines()) == 11988


@pytest.mark.gpu
@need_cli
def test_cli_run_valid():  # cli.run
    rc, out, _ = rst("run", "gen:path:4", "bfs", "--root", "0")
    assert rc == 0 and re.search(r"valid +true", out)


@pytest.mark.gpu
@need_cli
def test_cli_stats_depth():  # cli.stats
    rc, out, _ = rst("stats", "gen:grid:100:100")
    assert rc == 0 and re.search(r"depth +198", out)


@pytest.mark.gpu
@need_cli
def test_cli_bench_csv():  # cli.bench
    rc, out, _ = rst("bench", "gen:path:64", "--algo", "bfs")
    assert rc == 0
    assert "dataset,algorithm,n,m,root,median_ms,steps,work,tree_depth,components,valid" in out


@pytest.mark.gpu
@need_cli
def test_cli_dump_validate(tmp_path):  # cli.dump_validate
    dump = str(tmp_path / "dump.txt")
    rc, _, _ = rst("run", "gen:grid:12:9", "pr-rst", "--root", "5", "--dump-parents", dump)
    assert rc == 0
    rc, out, _ = rst("validate", "gen:grid:12:9", dump, "--root", "5")
    assert rc == 0 and "valid rooted spanning forest" in out


@pytest.mark.gpu
@need_cli
def test_cli_json():  # cli.json
    rc, out, _ = rst("run", "gen:star:100", "cc-euler", "--json")
    assert rc == 0 and '"valid": true' in out


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(ACC), reason="build/rst_acceptance not built")
def test_acceptance_binary():
    p = subprocess.run([ACC], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert p.stdout.count("PASS") == 9

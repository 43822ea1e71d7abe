"""tools/mag_cli.c: a plain C caller of the mag.h ABI.

CPU: it compiles against this repo's include/mag.h AND, when present, the
reference's own proj/include/mag.h (the drop-in claim), links
libmag_b200.so, runs the host-only subcommands, and fails loudly (exit 1,
MAG_ERR_INTERNAL) for a search without a GPU.  GPU: the search output is
the SPEC's byte-exact TSV.
"""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1405_5483_b200")
REF_INC = "/root/reference/proj/include"


def build(tmp_path, inc):
    exe = str(tmp_path / "mag_cli")
    subprocess.run(["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-Werror", "-I", inc,
                    os.path.join(ROOT, "tools", "mag_cli.c"), "-L", LIBDIR, "-lmag_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def run(exe, *args, **kw):
    return subprocess.run([exe, *args], capture_output=True, text=True, timeout=300, **kw)


@pytest.fixture(scope="module")
def cli(tmp_path_factory, mag):
    return build(tmp_path_factory.mktemp("cli"), os.path.join(ROOT, "include"))


def test_builds_against_reference_header(tmp_path, mag):
    if not os.path.isdir(REF_INC):
        pytest.skip("reference header not present (GPU box)")
    exe = build(tmp_path, REF_INC)
    assert run(exe).returncode == 2


def test_tune_and_gen(cli, tmp_path, port):
    out = run(cli, "tune", "--sigma", "4", "--r", "10000", "--m", "32")
    assert out.returncode == 0, out.stderr
    kv = dict(l.split("=") for l in out.stdout.split())
    want = port.tune(4, 10000, 32)
    assert int(kv["q"]) == want["q"] and int(kv["k"]) == want["k"]
    corpus = tmp_path / "c.txt"
    corpus.write_bytes(b"ACGTTGCAAGCT" * 100)
    out = run(cli, "gen", "--corpus", str(corpus), "--r", "5", "--m", "8", "--seed", "7")
    assert out.returncode == 0, out.stderr
    pats = out.stdout.encode().split(b"\n")[:-1]
    offs = port.sample_offsets(1200, 5, 8, 7)
    assert pats == [(b"ACGTTGCAAGCT" * 100)[o:o + 8] for o in offs]


def test_usage_and_errors(cli, tmp_path):
    assert run(cli).returncode == 2
    assert run(cli, "search", "--patterns", "/nonexistent", "--text", "/nonexistent").returncode == 2
    p = tmp_path / "p.txt"
    p.write_bytes(b"abba\nbbac\n")
    t = tmp_path / "t.txt"
    t.write_bytes(b"xabbacy")
    out = run(cli, "search", "--patterns", str(p), "--text", str(t), "--variant", "naive")
    assert out.returncode == 1 and "bad configuration" in out.stderr


def test_search_without_gpu_fails_loudly(cli, tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = tmp_path / "p.txt"
    p.write_bytes(b"abba\nbbac\n")
    t = tmp_path / "t.txt"
    t.write_bytes(b"xabbacy")
    out = run(cli, "search", "--patterns", str(p), "--text", str(t))
    assert out.returncode == 1 and "CUDA" in out.stderr


@pytest.mark.gpu
def test_search_tsv(cli, tmp_path, ref):
    p = tmp_path / "p.txt"
    p.write_bytes(b"abba\nbbac\n")
    t = tmp_path / "t.txt"
    t.write_bytes(b"xabbacy")
    for v in ("mag", "smag", "shiftor_og"):
        out = run(cli, "search", "--patterns", str(p), "--text", str(t), "--variant", v)
        assert out.returncode == 0, out.stderr
        assert out.stdout == "0\t1\n1\t2\n"
    t.write_bytes(b"")
    out = run(cli, "search", "--patterns", str(p), "--text", str(t))
    assert out.returncode == 0 and out.stdout == ""
    rng = np.random.default_rng(3)
    text = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, 200000)]
    pats = [text[s:s + 20].tobytes() for s in rng.integers(0, text.size - 20, 30)]
    p.write_bytes(b"\n".join(pats) + b"\n")
    t.write_bytes(text.tobytes())
    offs, pids = ref.ac(text, pats)
    want = "".join(f"{i}\t{o}\n" for o, i in zip(offs.tolist(), pids.tolist()))
    out = run(cli, "search", "--patterns", str(p), "--text", str(t), "--q", "3", "--k", "2",
              "--mapping", "balance", "--sigma-prime", "4")
    assert out.returncode == 0 and out.stdout == want
    out = run(cli, "search", "--patterns", str(p), "--text", str(t), "--count")
    assert out.stdout == f"{offs.size}\n"


BENCH_HEADER = ("dataset,variant,r,m,q,k,sigma_prime,mapping,mb_per_s,filter_reads,candidates,"
                "occurrences")  # BenchRow field list, in order


def test_bench_header_and_usage(cli, tmp_path):
    assert run(cli, "bench").returncode == 2
    assert run(cli, "bench", "--text", "/nonexistent").returncode == 2
    t = tmp_path / "t.txt"
    t.write_bytes(b"ACGT" * 100)
    assert run(cli, "bench", "--text", str(t), "--r", "x").returncode == 2
    assert run(cli, "bench", "--text", str(t), "--variant", "mag,bogus").returncode == 2
    out = run(cli, "bench", "--text", str(t), "--r", "2", "--m", "8")
    assert out.stdout.split("\n")[0] == BENCH_HEADER
    import torch
    if not torch.cuda.is_available():
        assert out.returncode == 1 and "CUDA" in out.stderr


@pytest.mark.gpu
def test_bench_matrix(cli, tmp_path, ref):
    """2 variants x 2 r x 1 m -> 4 rows; --check passes and every
    occurrences column equals the reference AC count for the same sample."""
    import paper_1405_5483_b200 as mag
    rng = np.random.default_rng(11)
    text = np.frombuffer(b"ACGT", np.uint8)[rng.integers(0, 4, 1 << 20)]
    t = tmp_path / "dna.txt"
    t.write_bytes(text.tobytes())
    out = run(cli, "bench", "--text", str(t), "--name", "dna1m", "--variant", "mag,shiftor_og",
              "--r", "10,1000", "--m", "16", "--seed", "5", "--reps", "2", "--check")
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().split("\n")
    assert lines[0] == BENCH_HEADER and len(lines) == 5
    for row in lines[1:]:
        f = row.split(",")
        assert f[0] == "dna1m" and f[1] in ("mag", "shiftor_og") and f[3] == "16"
        r = int(f[2])
        pats = mag.sample_patterns(text, r, 16, 5)
        offs, _ = ref.ac(text, pats)
        assert int(f[11]) == offs.size >= r  # every sampled pattern occurs at its source
        assert float(f[8]) > 0 and int(f[9]) > 0
    # --include-prep and reference-mode parameters: q/k/sigma'/mapping echoed
    out = run(cli, "bench", "--text", str(t), "--r", "100", "--m", "32", "--include-prep", "--check",
              "--q", "4", "--k", "1", "--sigma-prime", "4", "--mapping", "balance", "--reps", "1",
              "--variant", "smag")
    assert out.returncode == 0, out.stderr
    f = out.stdout.strip().split("\n")[1].split(",")
    assert f[1] == "smag" and f[4:8] == ["4", "1", "4", "balance"]

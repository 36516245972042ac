"""The C++ façade (include/trim_b200/ivf.hpp): it compiles against the C ABI,
against the reference's own types (when /root/reference is present), and on
a GPU its test program passes (tests/cpp/test_facade.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")
LIBDIR = os.path.join(ROOT, "paper_2508_17828_b200")
REF_INC = "/root/reference/proj/include"


def _build(out):
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"), SRC,
           "-L", LIBDIR, "-ltrim_b200", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_facade_builds(tmp_path):
    _build(str(tmp_path / "t"))


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_facade_adapts_reference_types(tmp_path):
    """from_reference() instantiates with the reference's own IvfIndex / VectorDataset /
    PruningProfile (compile-only: no GPU here)."""
    src = tmp_path / "adapt.cpp"
    src.write_text(
        '#include "trimsearch/ivf/ivf.hpp"\n#include "trim_b200/ivf.hpp"\n'
        "using namespace trimsearch;\n"
        "int run(const ivf::IvfIndex& ix, const VectorDataset& ds, const trim::PruningProfile& p, VectorView q) {\n"
        "  auto g = trim_b200::from_reference(ix, ds);\n"
        "  auto r = trim_b200::ivf::search_trim_ivf_knn(g, p, q, 10, 8);\n"
        "  auto s = trim_b200::ivf::search_trim_ivf_range(g, p, q, 1.0f, 8);\n"
        "  auto b = trim_b200::ivf::search_baseline_ivfpq(g, q, 10, 8, 100);\n"
        "  return int(r.ids.size() + s.ids.size() + b.ids.size());\n}\n")
    r = subprocess.run(["g++", "-std=c++20", "-c", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
                        str(src), "-o", str(tmp_path / "adapt.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_graph_facade_adapts_reference_types(tmp_path):
    """trim_b200::graph::from_reference() instantiates with the reference's own
    GraphIndex / LandmarkStore / VectorDataset / PruningProfile (compile-only)."""
    src = tmp_path / "adapt_graph.cpp"
    src.write_text(
        '#include "trimsearch/graph/search.hpp"\n#include "trim_b200/graph.hpp"\n'
        "using namespace trimsearch;\n"
        "int run(const graph::GraphIndex& g, const trim::LandmarkStore& lm, const VectorDataset& ds,\n"
        "        const trim::PruningProfile& p, VectorView q) {\n"
        "  auto gg = trim_b200::graph::from_reference(g, lm, ds);\n"
        "  auto r = trim_b200::graph::search_trim_knn(gg, p, q, 10, 64);\n"
        "  auto s = trim_b200::graph::search_trim_range(gg, p, q, 1.0f, 64);\n"
        "  return int(r.ids.size() + s.ids.size());\n}\n")
    r = subprocess.run(["g++", "-std=c++20", "-c", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
                        str(src), "-o", str(tmp_path / "adapt_graph.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_facade_program_on_gpu(tmp_path):
    exe = str(tmp_path / "t")
    _build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr

"""CPU-side checks of the boundary: libtsf.so loads and exports every symbol
include/tsf.h declares; the oracle and the product path share no code."""
import ast
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "tsf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsf_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    fns = header_functions()
    for f in ["tsf_create", "tsf_temporal_attn", "tsf_spatial_attn", "tsf_spacetime_block", "tsf_destroy"]:
        assert f in fns


def test_library_builds_loads_and_exports_header_symbols():
    from paper_2604_16590_b200 import build
    build.build()  # no-op when up to date; nvcc cross-compiles without a GPU
    import paper_2604_16590_b200 as tsf
    L = tsf.lib()
    for f in header_functions():
        assert hasattr(L, f), f"{f} declared in tsf.h but not exported"
    assert sorted(n for n, _, _ in tsf.SIGNATURES) == header_functions()


def test_binding_signatures_match_header_arity():
    import paper_2604_16590_b200 as tsf
    src = open(os.path.join(ROOT, "include", "tsf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    for name, _, args in tsf.SIGNATURES:
        m = re.search(rf"\b{name}\s*\(([^)]*)\)", src)
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), name


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2604_16590_b200 as tsf
    with pytest.raises(tsf.TsfError):
        tsf.Layer(4, 64, 2, 32)


def imports_of(path):
    names = set()
    for dirpath, _, files in os.walk(path):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        names |= {a.name.split(".")[0] for a in node.names}
                    elif isinstance(node, ast.ImportFrom) and node.module and node.level == 0:
                        names.add(node.module.split(".")[0])
    return names


def test_oracle_and_product_are_independent():
    assert "paper_2604_16590_b200" not in imports_of(os.path.join(ROOT, "oracle"))
    assert "oracle" not in imports_of(os.path.join(ROOT, "paper_2604_16590_b200"))
    assert "oracle" not in imports_of(os.path.join(ROOT, "synth"))
    assert "paper_2604_16590_b200" not in imports_of(os.path.join(ROOT, "synth"))
    for root, _, files in os.walk(os.path.join(ROOT, "paper_2604_16590_b200", "csrc")):
        for f in files:
            assert "oracle" not in open(os.path.join(root, f)).read().lower() or f.endswith(".md")


def test_distributed_create_rejects_mismatched_world_without_collectives():
    """Fault injection on the distributed boundary: a world size the shape cannot
    shard, a rank outside the world, or a simulated world beyond one box fail
    synchronously with TSF_ERR_CONFIG before any device work or NCCL collective
    (so a misconfigured rank cannot leave its peers waiting in a collective)."""
    import ctypes
    import paper_2604_16590_b200 as tsf
    L = tsf.lib()
    h = ctypes.c_void_p()
    uid = (ctypes.c_char * 128)()
    assert L.tsf_create_dist(6, 64, 2, 64, uid, 0, 4, ctypes.byref(h)) == tsf.TSF_ERR_CONFIG   # K % P
    assert b"divisible" in L.tsf_last_error(None)
    assert L.tsf_create_dist(8, 66, 2, 64, uid, 0, 4, ctypes.byref(h)) == tsf.TSF_ERR_CONFIG   # N % P
    assert L.tsf_create_dist(8, 64, 2, 64, uid, 4, 4, ctypes.byref(h)) == tsf.TSF_ERR_CONFIG   # rank >= world
    assert L.tsf_create_dist(8, 64, 2, 64, uid, -1, 4, ctypes.byref(h)) == tsf.TSF_ERR_CONFIG
    assert L.tsf_create_dist(8, 64, 2, 48, uid, 0, 4, ctypes.byref(h)) == tsf.TSF_ERR_UNSUPPORTED
    assert L.tsf_create_sim(8, 64, 2, 64, 16, 2, ctypes.byref(h)) == tsf.TSF_ERR_CONFIG       # P > 8
    assert L.tsf_create_sim(8, 64, 2, 64, 4, 3, ctypes.byref(h)) == tsf.TSF_ERR_CONFIG        # bad mode
    assert L.tsf_create_sim(6, 64, 2, 64, 4, 2, ctypes.byref(h)) == tsf.TSF_ERR_CONFIG        # K % P
    assert not h.value
    assert L.tsf_world_size(None) == -1
    assert L.tsf_sync(None, None, 0) == tsf.TSF_ERR_CONFIG

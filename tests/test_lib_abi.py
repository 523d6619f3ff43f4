"""CPU-side checks of the C ABI library: it loads, exports every symbol include/rec.h
declares, the ctypes struct layouts match the header, and without a GPU the library
refuses to run (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "rec.h")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rec_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2203_07424_b200 import binding
    return binding.lib()


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert "rec_model_create" in names and "rec_serve" in names and "rec_query" in names
    from paper_2203_07424_b200 import binding
    for n in names:
        assert hasattr(L, n), n
        assert n in binding.EXPORTS, f"{n} missing from binding.EXPORTS"
    so = os.path.join(ROOT, "paper_2203_07424_b200", "libhercules_rec.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rec_[a-z_0-9]+)", out))
    assert set(names) <= exported


def test_struct_layouts_match_header():
    # compile a tiny C program printing sizeof/offsetof of the header structs
    from paper_2203_07424_b200 import binding as b
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "rec.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu %zu\n", sizeof(rec_model_desc), offsetof(rec_model_desc, seed),
        offsetof(rec_model_desc, nccl_id), offsetof(rec_model_desc, l2_persist_bytes),
        offsetof(rec_model_desc, top_shift), offsetof(rec_model_desc, arch),
        offsetof(rec_model_desc, n_tasks));
 printf("%zu %zu %zu\n", sizeof(rec_serve_policy), sizeof(rec_serve_report), sizeof(rec_trace_row));
 printf("%zu %zu\n", offsetof(rec_serve_report, completed), offsetof(rec_serve_report, stable));
 return 0; }
'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        lines = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    a = [int(x) for x in lines[0].split()]
    assert a == [C.sizeof(b.rec_model_desc), b.rec_model_desc.seed.offset,
                 b.rec_model_desc.nccl_id.offset, b.rec_model_desc.l2_persist_bytes.offset,
                 b.rec_model_desc.top_shift.offset, b.rec_model_desc.arch.offset,
                 b.rec_model_desc.n_tasks.offset]
    p = [int(x) for x in lines[1].split()]
    assert p == [C.sizeof(b.rec_serve_policy), C.sizeof(b.rec_serve_report), W.TRACE_DTYPE.itemsize]
    r = [int(x) for x in lines[2].split()]
    assert r == [b.rec_serve_report.completed.offset, b.rec_serve_report.stable.offset]


def test_no_cpu_fallback_without_gpu(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2203_07424_b200 import RecModel, RecError
    with pytest.raises(RecError) as ei:
        RecModel(W.TINY)
    assert "REC_E_CUDA" in str(ei.value)


def test_invalid_args_rejected_before_device(L):
    from paper_2203_07424_b200 import RecModel, RecError
    with pytest.raises(RecError) as ei:
        RecModel(W.TINY.with_(bottom=(13, 64, 16)))        # bottom out != dim
    assert "REC_E_INVALID_ARG" in str(ei.value) and "dim" in str(ei.value)
    with pytest.raises(RecError) as ei:
        RecModel(W.TINY.with_(top=(64, 2)))
    assert "REC_E_INVALID_ARG" in str(ei.value)
    with pytest.raises(RecError) as ei:
        RecModel(W.TINY.with_(dim=30, bottom=(13, 64, 30)))
    assert "REC_E_UNSUPPORTED" in str(ei.value)


def test_nccl_unique_id(L):
    from paper_2203_07424_b200 import nccl_unique_id
    assert len(nccl_unique_id()) == 128


def test_oracle_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_2203_07424_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f
                assert not re.search(r"#include\s*[<\"].*oracle", src), f
                assert "import_module(\"oracle" not in src, f

"""The C-ABI library: loads on CPU, exports every symbol the header
declares, and the ctypes descriptor matches the C struct layout."""

import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from conftest import ROOT
from paper_1801_03589_b200 import _capi

HEADER = os.path.join(ROOT, "include", "nesa_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nesa_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_header_symbols():
    lib = _capi.load()
    names = declared_functions()
    assert set(names) == set(_capi.EXPORTED_SYMBOLS)
    for n in names:
        assert hasattr(lib, n), n
    assert lib.nesa_abi_version() == _capi.NESA_ABI_VERSION


def test_descriptor_layout_matches_header():
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "nesa_b200.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(nesa_plan_desc), offsetof(nesa_plan_desc, perm),
         offsetof(nesa_plan_desc, near_blob), offsetof(nesa_plan_desc, aux_sin),
         offsetof(nesa_plan_desc, leaf_end), offsetof(nesa_plan_desc, options),
         sizeof(nesa_exchange_desc), offsetof(nesa_exchange_desc, max_contrib),
         offsetof(nesa_exchange_desc, contrib));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(c, "w").write(prog)
        try:
            subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        except (OSError, subprocess.CalledProcessError):
            pytest.skip("no C compiler")
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split()
    D = _capi.NesaPlanDesc
    X = _capi.NesaExchangeDesc
    assert [int(x) for x in out] == [ctypes.sizeof(D), D.perm.offset, D.near_blob.offset,
                                     D.aux_sin.offset, D.leaf_end.offset, D.options.offset,
                                     ctypes.sizeof(X), X.max_contrib.offset, X.contrib.offset]


def test_create_rejects_bad_descriptor_without_gpu():
    lib = _capi.load()
    d = _capi.NesaPlanDesc()
    d.abi_version = 999
    h = ctypes.c_void_p()
    rc = lib.nesa_plan_create(ctypes.byref(d), 0, ctypes.byref(h))
    assert rc == _capi.NESA_ERR_INVALID
    assert b"ABI" in lib.nesa_last_error()
    with pytest.raises(ValueError):
        _capi.check(rc)

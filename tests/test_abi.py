"""The C-ABI library loads here (no GPU) and exports every symbol include/emb_a2a.h declares."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "emb_a2a.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(emb_a2a_\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n != "emb_a2a_allgather_fn"))


def test_header_declares_the_boundary():
    d = declared()
    for must in ("emb_a2a_init", "emb_a2a_register_tables", "emb_a2a_forward",
                 "emb_a2a_destroy", "emb_a2a_pool_local", "emb_a2a_set_option",
                 "emb_a2a_last_error"):
        assert must in d


def test_library_exports_every_declared_symbol():
    import paper_2305_06942_b200 as p
    lib = ctypes.CDLL(p.LIB_PATH)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared()) == set(p.EXPORTED)


def test_status_strings_and_abi_version_without_gpu():
    from paper_2305_06942_b200 import _lib
    assert _lib.lib.emb_a2a_abi_version() == 1
    assert _lib.status_string(7) == "EMB_A2A_ETIMEOUT"
    assert _lib.status_string(8) == "EMB_A2A_EINDEX"


def test_init_without_gpu_fails_cleanly():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2305_06942_b200 import _lib
    h = ctypes.c_void_p()
    cb = _lib.ALLGATHER_FN(lambda a, b, n, u: 0)
    rc = _lib.lib.emb_a2a_init(0, 1, 0, cb, None, ctypes.byref(h))
    assert rc == _lib.ECUDA and not h.value


def test_sm100a_sass_in_library():
    """The product library carries sm_100a SASS (cuobjdump lists the cubin's arch)."""
    import shutil
    import subprocess
    import paper_2305_06942_b200 as p
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        return
    out = subprocess.run([exe, "--list-elf", p.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_ag_gemm_library_exports_every_declared_symbol():
    """include/ag_gemm.h: every declared entry point is exported and bound."""
    import paper_2305_06942_b200 as p
    from paper_2305_06942_b200 import _lib
    src = open(os.path.join(ROOT, "include", "ag_gemm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(ag_gemm_\w+)\s*\(", src, flags=re.M))
    names.discard("ag_gemm_allgather_fn")
    assert {"ag_gemm_init", "ag_gemm_register", "ag_gemm_forward", "ag_gemm_destroy"} <= names
    lib = ctypes.CDLL(p.LIB_PATH)
    assert not [n for n in names if not hasattr(lib, n)]
    assert names == set(_lib.AG_EXPORTED)

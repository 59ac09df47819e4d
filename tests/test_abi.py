"""CPU checks of the C-ABI library: it builds, loads, and exports every entry
point include/unilite_b200.h declares (no compute without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "unilite_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(ul_[a-z0-9_]+)\s*\(",
                                 text, re.M)))


def test_header_declares_entry_points():
    names = declared_symbols()
    assert "ul_gae_f32" in names and "ul_ppo_plan_run" in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol():
    from paper_2605_30313_b200 import _lib

    lib = _lib.lib()
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, f"declared but not exported: {missing}"
    # and the ctypes prototypes only bind real symbols
    for n in _lib.exported_names():
        assert hasattr(lib, n)
    assert lib.ul_version() == 1


def test_header_declares_every_exported_symbol():
    """The header is the complete ABI: nothing is exported undeclared."""
    import subprocess

    so = ROOT / "paper_2605_30313_b200" / "libunilite_b200.so"
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True,
                         text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if l.strip()}
    undeclared = sorted(exported - set(declared_symbols()))
    assert not undeclared, f"exported but not declared in the header: {undeclared}"


def test_only_abi_symbols_exported():
    import subprocess

    so = ROOT / "paper_2605_30313_b200" / "libunilite_b200.so"
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True,
                         text=True).stdout
    syms = [l.split()[-1] for l in out.splitlines() if l.strip()]
    assert syms and all(s.startswith("ul_") for s in syms), syms


def test_struct_layouts_match_native():
    from paper_2605_30313_b200 import _lib

    assert ctypes.sizeof(_lib.OptCtl) == _lib.lib().ul_opt_ctl_bytes()
    d = _lib.NetDesc.of((235, 512, 256, 128, 12))
    assert _lib.lib().ul_net_param_count(ctypes.byref(d)) == \
        235 * 512 + 512 + 512 * 256 + 256 + 256 * 128 + 128 + 128 * 12 + 12 + 12
    from paper_2605_30313_b200.tensornet import Arch

    ln = Arch(input_dim=235, hidden_dims=(512, 256, 128), output_dim=12, layer_norm=True)
    dl = ln.desc()
    assert _lib.lib().ul_net_param_count(ctypes.byref(dl)) == ln.param_count == \
        ctypes.c_int64(_lib.lib().ul_net_param_count(ctypes.byref(d))).value + 2 * (512 + 256 + 128)


def test_product_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_30313_b200 import algos
    import numpy as np

    with pytest.raises(RuntimeError, match="CUDA device"):
        algos.gae(np.zeros((2, 2)), np.zeros((2, 2)), np.zeros((2, 2), bool),
                  np.zeros((2, 2), bool), np.zeros(2), 0.99, 0.95)


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2605_30313_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f

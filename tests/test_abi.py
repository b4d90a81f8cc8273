"""Host-side checks of the C-ABI boundary (-m "not gpu"): the library builds
for sm_100a, loads without a GPU and exports every entry point that
include/fae.h declares; the product path never touches the oracle."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fae.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fae_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2103_00686_b200 import build
    return build.build()


def test_header_declares_the_paper_calls():
    d = _declared()
    for name in ["fae_profile", "fae_threshold", "fae_classify", "fae_emb_fwd",
                 "fae_emb_bwd_update", "fae_sync_hot_grads"]:
        assert name in d


def test_library_exports_every_declared_symbol(libpath):
    import paper_2103_00686_b200 as fae
    L = fae.lib()
    for name in _declared():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (fae_[a-z0-9_]+)\b", out))
    assert set(_declared()) <= exported
    assert set(fae.EXPORTS) == set(_declared())


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_product_path_never_uses_oracle():
    pkg = os.path.join(ROOT, "paper_2103_00686_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert "oracle" not in s.replace("oracle/ (the oracle is an independent C file)", ""), f


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    import paper_2103_00686_b200 as fae
    monkeypatch.setattr(fae, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(fae, "_lib", None)
    with pytest.raises(ImportError):
        fae.lib()

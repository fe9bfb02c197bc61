"""The oracle and the CUDA path share no code and never import each other;
the seeded-input module holds none of the method's arithmetic."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
IMPORT = re.compile(r"^\s*(?:from|import)\s+([\w.]+)", re.M)


def _files(d, exts=(".py", ".cu", ".cuh", ".h", ".c", ".cpp")):
    for dp, _, fs in os.walk(os.path.join(ROOT, d)):
        for f in fs:
            if f.endswith(exts):
                yield os.path.join(dp, f)


def _code(text):
    return re.sub(r'""".*?"""|#[^\n]*|//[^\n]*|/\*.*?\*/', "", text, flags=re.S)


def test_product_never_imports_oracle():
    for f in _files("paper_2502_12665_b200"):
        mods = IMPORT.findall(open(f).read())
        assert not any(m.split(".")[0] in ("oracle", "synth", "tests") for m in mods), f
        assert "oracle" not in _code(open(f).read()), f


def test_oracle_never_imports_product():
    for f in _files("oracle"):
        mods = IMPORT.findall(open(f).read())
        assert not any(m.split(".")[0] in ("paper_2502_12665_b200", "synth", "torch") for m in mods), f


def test_synth_holds_no_method_arithmetic():
    for f in _files("synth"):
        code = _code(open(f).read()).lower()
        for banned in ("rope", "rotate", "argmin", "softmax", "topk", "lut", "cholesky", "oracle", "sincos"):
            assert not re.search(r"\b%s\w*" % banned, code), (f, banned)

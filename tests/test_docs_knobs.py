"""Every MOE_* environment knob the native library reads is listed in
DESIGN.md §9 (the table a maintainer uses to re-run an A/B)."""
import pathlib
import re

ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_every_native_knob_is_documented():
    src = "".join(p.read_text() for p in (ROOT / "paper_2303_06182_b200" / "csrc").glob("*.c*"))
    src += "".join(p.read_text() for p in (ROOT / "paper_2303_06182_b200" / "csrc").glob("*.h"))
    knobs = set(re.findall(r'getenv\("(MOE_[A-Z0-9_]+)"\)', src))
    knobs |= set(re.findall(r'late_trigger\("(MOE_[A-Z0-9_]+)"', src))
    design = (ROOT / "DESIGN.md").read_text()
    table = design[design.index("## 9. Environment knobs"):]
    missing = sorted(k for k in knobs if f"`{k}`" not in table)
    assert knobs and not missing, missing

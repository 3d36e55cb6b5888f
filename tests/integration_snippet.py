"""Helper: the reference-side binding module exactly as INTEGRATION.md shows it."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def snippet_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```python\n(.*?)```", text, flags=re.S)
    (src,) = [b for b in blocks if b.startswith("# sfw3d/_b200.py")]
    return src


def load_snippet() -> dict:
    ns: dict = {"__name__": "sfw3d._b200"}
    exec(compile(snippet_source(), "INTEGRATION.md:sfw3d/_b200.py", "exec"), ns)
    return ns

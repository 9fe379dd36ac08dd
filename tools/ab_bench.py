"""bench.py's pipelined measurement with a variant library (AB_LIB) -> one line."""
import json
import os
import subprocess
import sys

sys.path.insert(0, ".")
from paper_2503_16422_b200 import _lib  # noqa: E402

if os.environ.get("AB_LIB"):
    _lib.LIB_PATH = os.path.abspath(os.environ["AB_LIB"])
sys.argv = ["bench.py"] + sys.argv[1:] + ["--no-cpu-baseline", "--no-e2e", "--steps", "6"]
import io  # noqa: E402
import contextlib  # noqa: E402
import bench  # noqa: E402

buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    bench.main()
d = json.loads(buf.getvalue().strip().splitlines()[-1])
print(d["value"], d["stages_isolated_ms_per_frame"])

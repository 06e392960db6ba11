"""Build experimental variants of libqmb200.so (A/B of -DQM_EXP_* switches) into exp_lib/.

    python scripts/build_variants.py name1='-DQM_EXP_EPI=1' name2='-DQM_EXP_DEPHASE=2000' ...

Each variant is the same library compiled with extra nvcc flags; select one at run time with
QM_LIB_PATH=exp_lib/libqmb200_<name>.so. The in-tree default library is rebuilt afterwards.
"""
import os
import shutil
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2011_11762_b200 import _build  # noqa: E402

out = _build.ROOT / "exp_lib"
out.mkdir(exist_ok=True)
for arg in sys.argv[1:]:
    name, flags = arg.split("=", 1)
    os.environ["QM_NVCC_EXTRA"] = flags
    _build.build(force=True)
    shutil.copy(_build.LIB, out / f"libqmb200_{name}.so")
    print("built", name, flags, flush=True)
os.environ.pop("QM_NVCC_EXTRA", None)
_build.build(force=True)

"""Run the reference's OWN test suite (pkg/tests of /root/reference) against this package.

    python tools/ref_suite.py prepare      # here (the build container): stage the suite
    python tools/ref_suite.py run [-- pytest args]   # on the GPU box (gpurun)

`prepare` copies the reference's test files, unmodified, into baseline/_ref/ref_tests/ (git-ignored,
so no reference source enters the repository's history; not gpurun-ignored, so it travels to the
GPU box, where /root/reference does not exist) and writes a small shim package `itq3` under
baseline/_ref/itq3_shim/ whose modules re-export this package's implementation under the
reference's module names (itq3.codec -> paper_2603_27914_b200.codec, ...).  Two private helpers the
reference tests import directly (itq3.compute._rotated_recon / _ternary_blocks, test_compute.py:
117-152) are not part of the drop-in API; the shim takes them from the CPU oracle (test
infrastructure).  test_cli.py is left out: the CLI is out of scope.

`run` executes the staged suite with pytest; every compute call goes through libitq3.so on the GPU.
Expected: every test passes except the reference's own documented ablation check
(test_acceptance.py::test_12, which fails on the reference itself).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/pkg/tests"
STAGE = os.path.join(ROOT, "baseline", "_ref")
SKIP = {"test_cli.py"}

SHIM = {
    "__init__": "from paper_2603_27914_b200 import *  # noqa: F401,F403\n",
    "codec": "from paper_2603_27914_b200.codec import *  # noqa: F401,F403\n"
             "from paper_2603_27914_b200.codec import QuantConfig, QuantizedTensor, decode_block, dequantize_tensor, "
             "encode_block, quantize_tensor, read_container, write_container  # noqa: F401\n",
    "errors": "from paper_2603_27914_b200.errors import *  # noqa: F401,F403\n",
    "packing": "from paper_2603_27914_b200.packing import *  # noqa: F401,F403\n"
               "from paper_2603_27914_b200.packing import F16_NAN, PackedBlock, block_nbytes, decode_f16, "
               "deserialize_block, encode_f16, pack_ternary, serialize_block, unpack_ternary  # noqa: F401\n",
    "quantizer": "from paper_2603_27914_b200.quantizer import *  # noqa: F401,F403\n",
    "transform": "from paper_2603_27914_b200.transform import *  # noqa: F401,F403\n",
    "selfcheck": "from paper_2603_27914_b200.selfcheck import *  # noqa: F401,F403\n"
                 "from paper_2603_27914_b200.selfcheck import CheckResult, run_selfcheck  # noqa: F401\n",
    "compute": '''from paper_2603_27914_b200.compute import fused_matmul, fused_matvec  # noqa: F401
from paper_2603_27914_b200.evaluate import *  # noqa: F401,F403
from paper_2603_27914_b200.evaluate import (AblationRow, ErrorReport, ablate_block_size, eval_error,  # noqa: F401
                                            generate_weights, report_csv, report_json, rotation_benefit)

# private helpers of the reference's vectorised encoder (compute.py:172-218), imported directly by
# test_compute.py:117-152 -- not part of the drop-in API, so they come from the CPU oracle
from oracle import itq3_oracle as _O


def _ternary_blocks(y, cfg):
    recon, codes, clamp, _budget = _O.ternary_blocks(y, cfg.variant, cfg.symmetric, cfg.policy.kind,
                                                     cfg.policy.constant)
    return recon, codes, clamp, None


def _rotated_recon(blocks, cfg):
    import numpy as np

    y = _O.fwht(np.asarray(blocks, dtype=np.float64))
    recon_y, codes, clamp, d16 = _ternary_blocks(y, cfg)
    return _O.fwht(recon_y), y, codes, clamp, d16
''',
}

CONFTEST = '''import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "itq3_shim"))   # `import itq3` -> the shim
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..", "..")))  # the repo root
'''


def prepare() -> None:
    dst = os.path.join(STAGE, "ref_tests")
    shutil.rmtree(dst, ignore_errors=True)
    os.makedirs(dst)
    n = 0
    for f in sorted(os.listdir(REF_TESTS)):
        if f.endswith(".py") and f not in SKIP and f != "conftest.py":
            shutil.copy(os.path.join(REF_TESTS, f), dst)
            n += 1
    with open(os.path.join(dst, "conftest.py"), "w") as fh:
        fh.write(CONFTEST)
    shim = os.path.join(STAGE, "itq3_shim", "itq3")
    shutil.rmtree(shim, ignore_errors=True)
    os.makedirs(shim)
    for name, body in SHIM.items():
        with open(os.path.join(shim, name + ".py"), "w") as fh:
            fh.write(body)
    print(f"staged {n} reference test files in {dst}; shim package in {shim}")


def run(extra: list[str]) -> int:
    dst = os.path.join(STAGE, "ref_tests")
    if not os.path.isdir(dst):
        print("nothing staged: run `python tools/ref_suite.py prepare` in the build container first")
        return 2
    cmd = [sys.executable, "-m", "pytest", dst, "-q", "-p", "no:cacheprovider", "--rootdir", dst] + extra
    return subprocess.call(cmd, cwd=dst)


if __name__ == "__main__":
    if len(sys.argv) < 2 or sys.argv[1] not in ("prepare", "run"):
        print(__doc__)
        sys.exit(2)
    if sys.argv[1] == "prepare":
        prepare()
    else:
        extra = sys.argv[2:]
        if extra and extra[0] == "--":
            extra = extra[1:]
        sys.exit(run(extra))

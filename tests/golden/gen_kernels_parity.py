"""Golden outputs of the reference's own kernel bit-parity suite
(pkg/tests/test_kernels_parity.py:14-57), made by running the REFERENCE
(its compiled `native` backend, which that suite proves bit-identical to its
`python` backend) on exactly that suite's inputs: the same seeds, shapes and
draw order (reference core.make_rng / sample_standard_normal).  The GPU box
has no reference, so tests/test_gpu_reference_kernel_parity.py replays the
suite against these outputs with the CUDA backend in the `native` slot.

    NSNKV_REF_SRC=/tmp/refpkg/src python tests/golden/gen_kernels_parity.py
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, os.environ.get("NSNKV_REF_SRC", "/root/reference/pkg/src"))
sys.path.insert(0, str(HERE.parents[1]))

from nsnkv import kernels  # noqa: E402

from tests.golden.inputs import kernels_parity_inputs  # noqa: E402


def main():
    back = kernels.backends()
    impl = back.get("native", back["python"])
    print("reference backend:", "native" if "native" in back else "python")
    out = {}
    inp = kernels_parity_inputs()
    for d, x in inp["fwht"].items():
        out[f"fwht_{d}"] = impl.fwht_rows(x)
        assert np.array_equal(out[f"fwht_{d}"], back["python"].fwht_rows(x))
    for name, (vecs, entries, fold) in inp["match"].items():
        inv = kernels.entry_inv_norms(entries)
        idx, sg = impl.match_block(vecs, entries, inv, fold)
        out[f"match_idx_{name}"] = idx
        out[f"match_sgn_{name}"] = sg if sg is not None else np.zeros(0, np.uint8)
    np.savez_compressed(HERE / "kernels_parity.npz", **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()

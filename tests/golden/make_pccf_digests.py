"""PCCF golden digests made by the REFERENCE compiler (build container only).

For every golden case (tests/golden/*.npz, each block size) and for two
circuits too large to recompile with the reference at test time — a tied
HMM with 512 hidden states over 32 positions and this package's 3072-
variable HCLT of latent 64 — the sha256 of the reference's
``dumps_compiled(compile_circuit(g, cfg))`` bytes.  tests/test_pccf.py
compares this package's PCCF bytes against them.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_pccf_digests.py
"""
import hashlib
import json
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parents[1]))
sys.dont_write_bytecode = True

import make_golden as mg  # noqa: E402  (imports the reference)
from pcirc.compiler.cache import dumps_compiled  # noqa: E402

from _digest_cases import BIG  # noqa: E402


def main():
    sys.path.insert(0, str(HERE.parent))
    from _golden import cases, load
    out = {}
    for name in cases():
        rec = load(name)
        rg = mg.from_parts_ref(rec)
        for k in rec["ks"].tolist():
            c = mg.compile_circuit(rg, mg.CompileConfig(block_size=k))
            out[f"{name}/k{k}"] = hashlib.sha256(dumps_compiled(c)).hexdigest()
    for key, (build, k) in BIG.items():
        t0 = time.time()
        rg = mg.from_parts_ref(mg.graph_arrays(build()))
        c = mg.compile_circuit(rg, mg.CompileConfig(block_size=k))
        out[key] = hashlib.sha256(dumps_compiled(c)).hexdigest()
        print(key, f"{time.time() - t0:.1f}s", flush=True)
    (HERE / "pccf_digests.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()

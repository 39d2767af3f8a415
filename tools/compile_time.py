"""Host-side build times of a bench workload: structure generation,
compile_circuit (native core, or PCB_COMPILER=numpy) and the device-plan
tables (runtime/plan.py build_program), wall clock on this host:
    python tools/compile_time.py <workload> [--numpy]"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "hclt256"
    if "--numpy" in sys.argv:
        os.environ["PCB_COMPILER"] = "numpy"
    import bench
    from paper_2406_00766_b200 import structures as S
    from paper_2406_00766_b200.compiler import CompileConfig, compile_circuit
    from paper_2406_00766_b200.compiler import _native
    from paper_2406_00766_b200.runtime.plan import build_program
    w = bench.WORKLOADS[name]
    keys = ("kind", "num_vars", "hidden_dim", "num_categories", "seq_len", "vocab_size",
            "shape", "split_interval", "elementwise", "depth", "num_input_components",
            "num_repetitions", "tree")
    cfg = S.StructureConfig(seed=0, tied=True, **{k: w[k] for k in keys if k in w})
    t0 = time.perf_counter()
    g = S.build_structure(cfg)
    t1 = time.perf_counter()
    c = compile_circuit(g, CompileConfig(block_size=w["block"]), validate=False)
    t2 = time.perf_counter()
    build_program(c)
    t3 = time.perf_counter()
    print(json.dumps({"workload": name, "compiler": "native" if _native.lib() else "numpy",
                      "threads": os.cpu_count(), "edges": int(c.num_edges),
                      "structure_s": round(t1 - t0, 2), "compile_s": round(t2 - t1, 2),
                      "plan_tables_s": round(t3 - t2, 2)}))


if __name__ == "__main__":
    main()

"""Run a few bench steps of a workload (for ncu launch lists / kernel captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

import bench
from paper_2406_00766_b200.runtime import _lib
from paper_2406_00766_b200.runtime.buffers import allocate_buffers
from paper_2406_00766_b200.runtime.em import em_update_
from paper_2406_00766_b200.runtime.plan import device_plan


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "hclt256"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    w = bench.WORKLOADS[name]
    c = bench.build_circuit(w)
    B = w["batch"]
    plan = device_plan(c)
    bufs = allocate_buffers(c, B, plan=plan)
    x = torch.from_numpy(bench.synthetic_batches(c, w, B, 1, 0)[0]).cuda()
    s = _lib.stream_handle()
    pf = 0 if plan.info.get("prod_flows_optional") else bufs.prod_flows_full.data_ptr()
    _lib.call("pcb_plan_set_lean", plan.handle, 1)  # as runtime.step.TrainStep
    for _ in range(steps):
        _lib.call("pcb_transpose_batch_i32", plan.handle, s, B, bufs.ldb, x.data_ptr(),
                  bufs.xT.data_ptr())
        _lib.call("pcb_forward", plan.handle, s, B, bufs.ldb, bufs.xT.data_ptr(),
                  plan.theta.data_ptr(), bufs.values_full.data_ptr(), bufs.scratch_full.data_ptr(),
                  bufs.lroot.data_ptr(), bufs.work.data_ptr())
        _lib.call("pcb_backward", plan.handle, s, B, bufs.ldb, bufs.xT.data_ptr(),
                  plan.theta.data_ptr(), bufs.values_full.data_ptr(), bufs.flows_full.data_ptr(),
                  bufs.scratch_full.data_ptr(), bufs.flow_scratch_full.data_ptr(),
                  pf, bufs.f_params.data_ptr(),
                  bufs.work.data_ptr())
        em_update_(c, bufs.f_params, pseudocount=1e-6, step_size=0.01, check=False, plan=plan)
    torch.cuda.synchronize()
    print("done", name, steps)


if __name__ == "__main__":
    main()

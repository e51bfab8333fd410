"""5a with the scratch (direct tables included) in plain vs compressible device memory
(cuMemCreate + CU_MEM_ALLOCATION_COMP_GENERIC, via cuda-python; the library only sees
the pointer).  One JSON line per allocation kind: per-launch generate / scan / clear
ms (sequential and overlapped) and the graph-replay step."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda.bindings import driver as cu
import paper_2203_12878_b200 as mc
from workloads import config


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) == 2 else r


class CompressibleBuffer:
    def __init__(self, nbytes, dev=0):
        prop = cu.CUmemAllocationProp()
        prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = dev
        prop.allocFlags.compressionType = cu.CUmemAllocationCompType.CU_MEM_ALLOCATION_COMP_GENERIC
        gran = ck(cu.cuMemGetAllocationGranularity(prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
        self.size = (nbytes + gran - 1) // gran * gran
        self.h = ck(cu.cuMemCreate(self.size, prop, 0))
        got = ck(cu.cuMemGetAllocationPropertiesFromHandle(self.h))
        self.compressed = int(got.allocFlags.compressionType)
        self.va = ck(cu.cuMemAddressReserve(self.size, 0, 0, 0))
        ck(cu.cuMemMap(self.va, self.size, 0, self.h, 0))
        ad = cu.CUmemAccessDesc()
        ad.location = prop.location
        ad.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        ck(cu.cuMemSetAccess(self.va, self.size, [ad], 1))
        self.__cuda_array_interface__ = {"shape": (self.size,), "typestr": "|u1", "data": (int(self.va), False),
                                         "version": 3, "strides": None}


def run(p, scratch, tag, extra):
    out = {"scratch": tag, **extra}
    for ovl in (False, True):
        p.check_races(scratch=scratch, overlap=ovl)
        r = p.check_races(scratch=scratch, overlap=ovl, profile=True)
        ks = {k: round(v["ms"] / max(1, v["launches"]), 4) for k, v in r.kernels.items() if v["launches"]}
        out["overlap" if ovl else "alone"] = {"per_launch_ms": ks, "step_ms": round(r.device_ms, 3)}
    ms = [p.check_races(scratch=scratch).device_ms for _ in range(6)]
    out["graph_step_ms"] = round(min(ms), 3)
    out["G_acc_s"] = round(2**34 / min(ms) / 1e6, 1)
    print(json.dumps(out), flush=True)


torch.cuda.init()
inst = config("5a")
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
need = p.scratch_bytes()
plain = torch.empty(need, dtype=torch.uint8, device="cuda")
run(p, plain, "cudaMalloc", {})
buf = CompressibleBuffer(need)
comp = torch.as_tensor(buf, device="cuda")
assert comp.data_ptr() == int(buf.va)
run(p, comp, "compressible", {"granted": buf.compressed})
run(p, plain, "cudaMalloc", {})
run(p, comp, "compressible", {"granted": buf.compressed})

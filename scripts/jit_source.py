"""Print the NVRTC-specialised generate source of one chunk of a config
(MAPC_DEBUG_JIT_MODE=0 keys / 1 direct / 2 filter), e.g. to inspect it or to
compile it with nvcc -cubin -Xptxas -v for the register count."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_12878_b200 as mc
from workloads import config

inst = config(sys.argv[1] if len(sys.argv) > 1 else "5a")
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 0
p = mc.MapProgram(inst.src, inst.grid, inst.block, inst.params)
f = mc._lib.map_debug_jit_source
f.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_char_p, ctypes.c_size_t]
f.restype = ctypes.c_size_t
buf = ctypes.create_string_buffer(1 << 22)
f(p._h, 0, chunk, buf, 1 << 22)
print(buf.value.decode())

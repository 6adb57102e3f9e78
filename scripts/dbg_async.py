import sys, ctypes, numpy as np
sys.path.insert(0, '.')
from paper_2002_12115_b200 import native as N
from paper_2002_12115_b200.apps import himeno
name = sys.argv[1]; nn = int(sys.argv[2])
sz = himeno.size(name)
a = N.Context(0, sz.I, sz.J, sz.K); b = N.Context(0, sz.I, sz.J, sz.K)
a.init_device()
lib = a.lib
nbytes = sz.I * sz.J * sz.K * 4
host = {}
for f in N.FIELDS:
    ptr = lib.hp_host_alloc(nbytes)
    host[f] = np.ctypeslib.as_array((ctypes.c_float * (nbytes // 4)).from_address(ptr)).reshape(sz.I, sz.J, sz.K)
    host[f][...] = a.read_field(f, 1)
outs = []
for _ in range(2):
    ptr = lib.hp_host_alloc(nbytes)
    outs.append(np.ctypeslib.as_array((ctypes.c_float * (nbytes // 4)).from_address(ptr)).reshape(sz.I, sz.J, sz.K))
gs = a.jacobi_host(host, nn, 1, outs[0]); ref = outs[0].copy()
print("serial", gs)
gb = b.jacobi_host(host, nn, 1, outs[1]); print("serial b", gb, np.array_equal(outs[1], ref))
for trial in range(2):
    a.jacobi_host_async(host, nn, 1, outs[0]); b.jacobi_host_async(host, nn, 1, outs[1])
    ga_, gb_ = a.sync(), b.sync()
    print("async", ga_, gb_, np.array_equal(outs[0], ref), np.array_equal(outs[1], ref),
          np.abs(outs[0]-ref).max(), np.abs(outs[1]-ref).max())

"""Same-box library bar: CUB radix sort (56 significant bits) + unique on the
bench's N2 batch keys, next to dedup_global on the same keys."""
import ctypes, os, subprocess, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
so = os.path.join(ROOT, "tools", "libcub_dedup.so")
subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                       "-Xcompiler", "-fPIC", "-o", so, os.path.join(ROOT, "tools", "cub_dedup.cu")])
L = ctypes.CDLL(so)
import paper_2604_15768_b200 as P, synth
wl, ints, par = synth.workload_inputs("n2", n_parents=1_000_000)
ctx = P.Context(0)
sp = P.Space(wl.m, 7, 7); di = P.DeviceIntegrals(ints.h, ints.eri)
shard = ctx.dedup_global(sp, torch.from_numpy(par).cuda())
rec = ctx.gen_coupled(sp, shard[:500_000], di, 0.0, with_src=False)
keys = rec.keys[:rec.count].reshape(-1)
n = keys.numel()
for _ in range(2):
    u = ctx.dedup_global(sp, rec.keys)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); u = ctx.dedup_global(sp, rec.keys); e1.record(); torch.cuda.synchronize()
ours = e0.elapsed_time(e1)
nu = u.shape[0]
del u, rec.hij
sorted_ = torch.empty_like(keys); out = torch.empty_like(keys)
nout = ctypes.c_longlong(); ms1 = ctypes.c_float(); ms2 = ctypes.c_float()
for _ in range(2):
    rc = L.cub_dedup(ctypes.c_void_p(keys.data_ptr()), ctypes.c_longlong(n), 56, ctypes.c_void_p(sorted_.data_ptr()),
                     ctypes.c_void_p(out.data_ptr()), ctypes.byref(nout), ctypes.byref(ms1), ctypes.byref(ms2))
print(f"N2 batch: {n} keys -> {nu} unique.  dedup_global: {ours:.2f} ms.  CUB SortKeys(56 bits) + Unique: "
      f"{ms1.value + ms2.value:.2f} ms ({ms1.value:.2f} + {ms2.value:.2f}), {nout.value} unique, rc={rc}")

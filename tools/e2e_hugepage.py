"""e2e host pipeline with pinned buffers from different allocators:
torch pin_memory vs THP-backed (madvise(MADV_HUGEPAGE)) memory registered with
cudaHostRegister."""
import mmap, sys, statistics
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2501_07535_b200 import kernels as K
from paper_2501_07535_b200.params import find_ntt_params
print(open('/sys/kernel/mm/transparent_hugepage/enabled').read().strip(), open('/sys/kernel/mm/transparent_hugepage/defrag').read().strip())
N, B = 1 << 16, 64
plan = K.get_plan(256, find_ntt_params(256, N))
nbytes = B * N * 32
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3 / 128
_keep = []
def huge(nb):
    m = mmap.mmap(-1, nb, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    a = np.frombuffer(m, dtype=np.int64).reshape(-1, 4)
    a[:] = 0
    rc = torch.cuda.cudart().cudaHostRegister(a.ctypes.data, nb, 0)
    _keep.append(m)
    return torch.from_numpy(a)
src = torch.randint(0, 1 << 59, (B * N, 4), dtype=torch.int64)
for trial in range(3):
    a = torch.empty((B * N, 4), dtype=torch.int64, pin_memory=True); a.copy_(src)
    b = torch.empty((B * N, 4), dtype=torch.int64, pin_memory=True)
    print("torch pinned", round(t(lambda: plan.host_transform(a, b, mode="forward_inverse", word_bits=64, ref_words=4)), 2), flush=True)
    h1 = huge(nbytes); h1.copy_(src); h2 = huge(nbytes)
    print("THP + cudaHostRegister", round(t(lambda: plan.host_transform(h1, h2, mode="forward_inverse", word_bits=64, ref_words=4)), 2), flush=True)

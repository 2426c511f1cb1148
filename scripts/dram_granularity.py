"""DRAM bytes moved by random 32 B and 64 B record gathers (run under ncu --cache-control all):
how many bytes one random 32 B sector read costs on this GPU, with the default L2 fetch
granularity and with cudaLimitMaxL2FetchGranularity lowered (argv[1] bytes, 0 = default)."""
import sys
import torch
g = int(sys.argv[1]) if len(sys.argv) > 1 else 0
torch.cuda.init()
if g:
    from cuda.bindings import runtime as rt
    err, = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity, g)
    print("set limit", g, err, rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity))
N = 1 << 26  # 2 GiB of 32 B rows: far larger than L2
x = torch.empty((N, 4), dtype=torch.float64, device="cuda").uniform_()
y = torch.empty((N // 2, 8), dtype=torch.float64, device="cuda").uniform_()
idx = torch.randint(0, N, (1 << 20,), device="cuda")
idx2 = torch.randint(0, N // 2, (1 << 20,), device="cuda")
a = x.index_select(0, idx)   # 1 Mi random 32 B rows
b = y.index_select(0, idx2)  # 1 Mi random 64 B rows
torch.cuda.synchronize()
print(a.sum().item() + b.sum().item())

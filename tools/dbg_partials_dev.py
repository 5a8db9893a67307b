import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2408_12057_b200 import abi, capi, distributed
tg = abi.scale_gaussian(1.0, 2.0, 1000); k = abi.kernel(abi.KERNEL_RWMH, (0.1,1.0,10.0), 1)
n = 1 << 21
dev = torch.device("cuda", 0); stream = torch.cuda.current_stream(dev)
ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32, 0, 0, stream.cuda_stream)
betas = np.array([0.0, 1.0]); T = 1
ranges = distributed.chunk_partition(n, 2)
print(ranges)
parts = []
for (p0, p1) in ranges:
    c = distributed.chunks_of((p0, p1))
    loc = torch.zeros((c, T + 1, 4, 2), dtype=torch.float64, device=dev)
    capi.sais_partials_dev(tg, k, betas, n, p0, p1, loc.data_ptr(), seed=1, round=1, exec_=ex)
    host = capi.sais_partials(tg, k, betas, n, p0, p1, seed=1, round=1, exec_=ex)
    print(p0, p1, c, float(loc[0,1,1,0]), float(loc[0,1,1,1]), host[0,1,1], np.array_equal(loc.cpu().numpy(), host))
    parts.append(loc)
allp = torch.cat(parts).contiguous()
rep = capi.fold_partials_dev(allp.data_ptr(), allp.shape[0], T, n, exec_=ex)
print(rep["log_z_hat"], capi.fold_partials(allp.cpu().numpy(), n)["log_z_hat"])

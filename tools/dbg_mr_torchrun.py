import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_12057_b200 import abi, capi, distributed
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
stream = torch.cuda.current_stream()
ex = abi.execopts(abi.RNG_PHILOX, abi.PREC_FP32, device=0, stream=stream.cuda_stream)
tg = abi.scale_gaussian(1.0, 2.0, 1000); k = abi.kernel(abi.KERNEL_RWMH, (0.1,1.0,10.0), 1)
capi.peak_normals(0, 148 * 8, 1 << 10)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
try:
    r = distributed.run_sais(tg, k, 1 << 21, 4, 1, ex, rank, world, device="cpu")
    print(rank, r["log_z_hat"], flush=True)
except Exception as e:
    print(rank, "ERR", e, flush=True)
    import traceback; traceback.print_exc()
dist.destroy_process_group()

import sys; sys.path.insert(0, "/root/repo")
import torch
from paper_2605_02568_b200 import api
from paper_2605_02568_b200.engine import Engine
e = Engine(0)
S, k = 262144, 1024
q = e.gen_normal_bf16(S*64*128, 128**-0.5, 1, 1); kc = e.gen_normal_bf16((S//4)*128, 128**-0.5, 1, 2); w = e.gen_normal_f32(S*64, (64*128)**-0.5, 1, 3)
dims = api.ProblemDims.create(1, S, 4, 64, 128, k)
cfg = api.DriverConfig(tile=api.TileConfig(2048, S//4))
api.run_chunked_device(q, kc, w, dims, cfg, [S-2048, 131072, 32768])
torch.cuda.synchronize()
print("done")

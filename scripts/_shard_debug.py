import sys, subprocess, itertools
code = r'''
import sys, torch
sys.path.insert(0, "/root/repo")
import paper_1704_08657_b200 as dwt
from paper_1704_08657_b200 import strips as S
from paper_1704_08657_b200.synth import random_image
W, world, L, iters, mode = [int(x) for x in sys.argv[1:6]]
plan = dwt.Plan("cdf97", "nonseparable-lifting", optimized=True)
Hs = W // world
img = random_image(W, W, 1, device="cuda")
strips = [img[r * Hs:(r + 1) * Hs].contiguous() for r in range(world)]
full = plan.forward_mallat(img, L)
torch.cuda.synchronize()
streams = [torch.cuda.Stream() for _ in range(world)]
if mode == 0:
    shards = [S.Shard(plan, W, Hs, L, r, world) for r in range(world)]
    S.connect_ring(shards)
    for it in range(iters):
        outs = [sh.forward_mallat(s, stream=st) for sh, s, st in zip(shards, strips, streams)]
else:
    for it in range(iters):
        outs = S.forward_mallat_sharded(plan, strips, L, streams=streams)
torch.cuda.synchronize()
print("OK", torch.equal(S.assemble_mallat(outs, L), full.cpu()))
'''
open("/tmp/sd.py", "w").write(code)
for cfg in [(512,3,5,2,0),(512,3,5,3,0),(512,3,8,2,0),(2048,2,5,2,0),(2048,2,8,2,0),(4096,2,8,1,0),(4096,2,8,2,0),(4096,4,8,2,1),(16384,4,8,3,1)]:
    r = subprocess.run(["timeout","60",sys.executable,"/tmp/sd.py"]+[str(c) for c in cfg], capture_output=True, text=True)
    print(cfg, r.returncode, (r.stdout.strip() or r.stderr.strip().splitlines()[-1] if r.stderr.strip() else "")[-120:], flush=True)

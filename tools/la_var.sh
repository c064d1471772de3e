for d in 0 1 3; do echo "dbg=$d"; TTSVD_BLK_DBG=$d python - <<'PY'
import torch, time, sys
sys.path.insert(0,'.')
import paper_2102_00104_b200 as tt
g=torch.Generator(device='cuda').manual_seed(1)
X=torch.rand(256,1<<20,dtype=torch.float64,device='cuda',generator=g).t()
for i in range(3):
    torch.cuda.synchronize(); t=time.perf_counter(); R=tt.tsqr(X); torch.cuda.synchronize(); print(f"{1e3*(time.perf_counter()-t):.2f} ms")
PY
done

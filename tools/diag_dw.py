import ctypes, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1503_02852_b200 import _lib
L = _lib.lib()
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
def dw(e, y, mode):
    k, m = e.shape; n = y.shape[1]
    te = torch.tensor(e, dtype=torch.float32, device='cuda'); ty = torch.tensor(y, dtype=torch.float32, device='cuda')
    tg = torch.full((m, n), float('nan'), device='cuda')
    _lib.check(L.rgb_gemm_dw(ctypes.c_void_p(te.data_ptr()), ctypes.c_void_p(ty.data_ptr()), ctypes.c_void_p(tg.data_ptr()), m, n, k, ctypes.c_float(1.0), mode, st))
    torch.cuda.synchronize()
    return tg.cpu().numpy()
np.set_printoptions(linewidth=200, precision=2, suppress=True)
K, M, N = 32, 128, 256
rng = np.random.default_rng(0)
e = rng.uniform(-1, 1, size=(K, M)); y = rng.uniform(-1, 1, size=(K, N))
g = dw(e, y, 2); ref = e.T @ y
print('nan', np.isnan(g).sum(), 'absmax', np.nanmax(np.abs(g)), 'ref absmax', np.abs(ref).max())
# structured: E = onehot rows: E[k, m] = 1 if m == k  -> G[m, n] = Y[m, n] for m < K
e2 = np.zeros((K, M)); e2[np.arange(K), np.arange(K)] = 1.0
y2 = np.arange(K)[:, None] * 1000.0 + np.arange(N)[None, :]
g2 = dw(e2, y2, 2)
print('G rows 0..9, cols 0..9:\n', g2[:10, :10])
print('G rows 30..34, cols 0..6:\n', g2[30:35, :7])
nz = np.argwhere(np.abs(g2) > 0)
print('nonzero count', len(nz), 'first', nz[:10])
# with mode 1 for reference
print('simt ok', np.abs(dw(e, y, 1) - ref).max())

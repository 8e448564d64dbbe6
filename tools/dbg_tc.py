import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2303_03279_b200 import compute_connectivity
z=np.load('tests/golden/rect_accept.npz')
x=torch.tensor(z['epochs'],device='cuda')
for ms in (["COHY"],["COH"],["PLV"],["COHY","COH"],["COHY","PLV"],["COH","PLV"],["COHY","COH","PLV"]):
    out,plan=compute_connectivity(x,int(z['nfft']),int(z['lo']),int(z['hi']),metrics=ms)
    torch.cuda.synchronize()
    res=[]
    for m in ms:
        got=out[m]['bins'].cpu().numpy().T; want=z['bins_'+m]
        gb=out[m]['band'].cpu().numpy(); wb=z['cband_COHY'] if m=='COHY' else z['band_'+m]
        res.append((m, float(np.nanmax(np.abs(got-want))), int(np.isnan(got).sum()), float(np.nanmax(np.abs(gb-wb)))))
    print(ms, res)

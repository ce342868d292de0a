import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle as O, paper_2506_08018_b200 as K
def run(kb, vb, D, H, chunks, seed, G=1, rows=1):
    dev = K.KVLayerCache(K.LayerQuantConfig(0, kb, vb, 0.2, 0.2, 32), 1, H, D, capacity_tokens=sum(chunks)+16)
    ora = O.CacheOracle(kb, vb, 0.2, 0.2, 32, 1, H, D)
    for i, t in enumerate(chunks):
        k = O.random_h16(seed + 2*i, (1, H, t, D)); v = O.random_h16(seed + 2*i + 1, (1, H, t, D))
        dev.append(k, v); ora.append(k, v)
    q = O.random_h16(seed + 77, (1, H * G, rows, D))
    ks, vs = ora.snapshot()
    qr = q.reshape(1, H, G * rows, D)
    o64, cs64 = O.attend_f64(qr, ks, vs)
    r = K.attend(torch.from_numpy(q).cuda(), dev)
    e = np.abs(r.output.cpu().numpy() - o64.reshape(q.shape)).max() / np.abs(vs).max()
    l1 = float(np.abs(np.einsum("bhtd,bhjd->bhtj", qr.astype(np.float64), ks.astype(np.float64))).sum() / np.sqrt(D))
    print(f"K{kb}V{vb} D{D} H{H} T{sum(chunks)} G{G} rows{rows}: e64={e:.2e} cs_err/l1={abs(r.scores_checksum-cs64)/l1:.2e}")
for D in (64, 128):
    for kb, vb in ((2,2),(4,4),(3,4),(2,4)):
        run(kb, vb, D, 2, [300, 1, 1, 40], 5)
run(2, 2, 128, 4, [2000] + [1]*30, 7)
run(2, 2, 128, 4, [2000] + [1]*30, 7, G=4)

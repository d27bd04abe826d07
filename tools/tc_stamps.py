"""Phase timeline of the first factor launch of k_leaf_apply_tc (variant built with -DKS_TC_TIMING=1).
Usage (GPU box): python tools/tc_stamps.py paper_1312_1869_b200/variants/tctime.so"""
import ctypes as C
import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib_path = os.path.join(ROOT, "paper_1312_1869_b200", "libks_b200.so")
shutil.copy(lib_path, "/tmp/ks_keep.so")
shutil.copy(sys.argv[1], lib_path + ".tmp")
os.replace(lib_path + ".tmp", lib_path)   # a new inode: never rewrite a mapped library in place
try:
    import torch
    import paper_1312_1869_b200 as ks
    os.environ["KS_TSQR_GRAPH"] = "0"
    dev = torch.device("cuda:0")
    Y = torch.randn(262144, 512, device=dev)
    plan = ks.TsqrPlan(262144, 512, 8, dev)
    plan.factor(Y, want_q=False)
    torch.cuda.synchronize()
    n = 1 << 20
    buf = (C.c_ulonglong * n)()
    assert ks.lib().ks_debug_tc_stamps(buf, n) == 0
    st = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 32, 8)[:264].astype(np.int64)   # [cta][item][slot]
    valid = st[:, :, 0] > 0
    t0 = st[valid][:, 0].min()
    names = ["p1", "w2", "p2wait_d", "p2wait_x", "p2blk0", "p2rest"]
    d = []
    for cta in range(st.shape[0]):
        for it in range(32):
            if not valid[cta, it]:
                continue
            s = st[cta, it]
            d.append([s[1] - s[0], s[2] - s[1], s[3] - s[2], s[4] - s[3], s[5] - s[4], s[6] - s[5]])
    d = np.array(d) / 1e3
    print(f"items {len(d)}; per-item mean (us): " + "  ".join(f"{n} {v:.2f}" for n, v in zip(names, d.mean(0))))
    print(f"item total mean {d.sum(1).mean():.2f} us; launch span {(st[valid][:, 6].max() - t0) / 1e3:.1f} us")
    w = np.frombuffer(buf, dtype=np.uint64)[1 << 19:(1 << 19) + 264 * 64].reshape(264, 32, 2).astype(np.int64)
    wv = w[valid]
    print(f"pass-1 waits per item (us): conv-slot / MMA done + drain {wv[:, 0].mean() / 1e3:.2f}, ring full {wv[:, 1].mean() / 1e3:.2f}")
    x = np.frombuffer(buf, dtype=np.uint64)[3 << 18:(3 << 18) + 264 * 128].reshape(264, 32, 4).astype(np.int64)[valid]
    print(f"pass-1 work per item (us): A conversion {x[:, 0].mean() / 1e3:.2f}, B conversion {x[:, 1].mean() / 1e3:.2f}, "
          f"fences + arrive {x[:, 2].mean() / 1e3:.2f}")
    print("items per CTA:", np.bincount(valid.sum(1))[np.bincount(valid.sum(1)) > 0], "(counts of CTAs by items)")
finally:
    shutil.copy("/tmp/ks_keep.so", lib_path + ".tmp")
    os.replace(lib_path + ".tmp", lib_path)

"""numpy restatement of the device-side synthetic V (kernels.cuh philox_normal2):
Philox4x32-10 keyed by (seed, global row, column pair) + Box-Muller. Test helper."""
import numpy as np


def philox_v(nd, nt, rank, seed):
    """numpy restatement of the device Philox4x32-10 + Box-Muller V (kernels.cuh)."""
    n = nd * nt
    gi = np.repeat(np.arange(n, dtype=np.uint64), (rank + 1) // 2)
    cp = np.tile(np.arange((rank + 1) // 2, dtype=np.uint64), n)
    M32 = np.uint64(0xFFFFFFFF)
    c = [gi & M32, gi >> np.uint64(32), cp & M32, cp >> np.uint64(32)]
    k0, k1 = np.uint64(seed & 0xFFFFFFFF), np.uint64(seed >> 32)
    for _ in range(10):
        p0 = np.uint64(0xD2511F53) * c[0]
        p1 = np.uint64(0xCD9E8D57) * c[2]
        c = [(p1 >> np.uint64(32)) ^ c[1] ^ k0, p1 & M32, (p0 >> np.uint64(32)) ^ c[3] ^ k1, p0 & M32]
        k0 = (k0 + np.uint64(0x9E3779B9)) & M32
        k1 = (k1 + np.uint64(0xBB67AE85)) & M32
    a = (c[0] << np.uint64(32)) | c[1]
    b = (c[2] << np.uint64(32)) | c[3]
    u1 = ((a >> np.uint64(11)).astype(np.float64) + 1.0) / 9007199254740992.0
    u2 = (b >> np.uint64(11)).astype(np.float64) / 9007199254740992.0
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.stack([r * np.cos(2 * np.pi * u2), r * np.sin(2 * np.pi * u2)], axis=1).reshape(n, -1)
    return z[:, :rank]

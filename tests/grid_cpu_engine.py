"""TEST INFRASTRUCTURE: a CPU engine for paper_1402_3661_b200.grid backed by
the oracle, so the grid's exchange schedule runs under gloo without a GPU."""
import numpy as np
import torch

import oracle as O
from helpers import to_oracle


class _Buf:
    def __init__(self, n, L):
        self.tensor = torch.zeros((n, L), dtype=torch.int32)


class OracleEngine:
    def __init__(self, block):
        self.orc = to_oracle(block)
        self.ell = block.mod.ell
        self.L = block.mod.limbs
        self.W = self.L

    def alloc(self, n):
        return _Buf(n, self.L)

    def scratch(self, n):
        return torch.zeros((n, self.L), dtype=torch.int32)

    def _np(self, t):
        return t.numpy().view(np.uint32)

    def spmv(self, src, dst):
        dst.tensor.copy_(torch.from_numpy(self.orc.spmv_limbs(self._np(src.tensor)).view(np.int32)))

    def add_mod(self, dst_tensor, srcs):
        tot = [0] * dst_tensor.shape[0]
        for t in srcs:
            for k, v in enumerate(O.limbs_to_ints(self._np(t))):
                tot[k] += v
        out = O.ints_to_limbs([x % self.ell for x in tot], self.L)
        dst_tensor.copy_(torch.from_numpy(out.view(np.int32)))

    def upload(self, buf, limbs):
        buf.tensor.copy_(torch.from_numpy(np.ascontiguousarray(limbs, dtype=np.uint32).view(np.int32)))

    def download(self, buf):
        return self._np(buf.tensor).copy()

    def read_rows(self, buf, rows):
        return self._np(buf.tensor)[list(rows)].copy() if len(rows) else np.zeros((0, self.L), np.uint32)

    def sync(self):
        pass

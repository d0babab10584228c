"""TEST INFRASTRUCTURE: a CPU stand-in for ep.CudaRank whose local compute is
the C oracle (oracle/moe_oracle.c), so the expert-parallel orchestration in
paper_2211_10017_b200/ep.py (counts, splits, all-to-all-v, regroup, combine)
can be exercised with gloo on CPU.  Never used by the product path."""
import numpy as np
import torch

from oracle.oracle import Oracle


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.float16).copy())


class OracleRank:
    def __init__(self, lw, e0, el, bits=4, q=None):
        self.o = Oracle()
        self.lw, self.e0, self.el, self.bits = lw, e0, el, bits
        self.E, self.d = lw.E, lw.d
        sl = slice(e0, e0 + el)
        if bits == 16:
            self.w = dict(w1=lw.w1[sl], w2=lw.w2[sl])
        else:
            q1, s1, q2, s2 = q
            nb1 = lw.d * lw.f // (2 if bits == 4 else 1)
            nb2 = lw.f * lw.d // (2 if bits == 4 else 1)
            self.w = dict(q1=q1[e0 * nb1:(e0 + el) * nb1], s1=s1[sl], q2=q2[e0 * nb2:(e0 + el) * nb2],
                          s2=s2[sl])
        self.b1, self.b2 = lw.b1[sl], lw.b2[sl]

    def route(self, x, fin, k):
        x = x.numpy().view(np.float16)
        T = x.shape[0]
        self.fin = np.zeros(T, np.uint8) if fin is None else fin.numpy().astype(np.uint8)
        xn = self.o.layer_norm(x, self.lw.ln_g, self.lw.ln_b)
        ex, sc = self.o.gate_topk(self.o.gate_logits(xn, self.lw.gw, self.lw.gb), k)
        self.scale = sc.view(np.float16)
        perm, inv, offs, act = self.o.routing_plan(ex, self.fin, self.E)
        self.inv, self.k = inv, k
        self.xp = xn[perm // k]
        self.y = np.zeros_like(self.xp)
        return offs.astype(np.int64)

    def sorted_rows(self, n):
        return _t(self.xp[:n])

    def y_rows(self, n):
        # a tensor aliasing the sorted-y buffer: the reverse all-to-all lands in it
        return torch.from_numpy(self.y[:n].view(np.int16)).view(torch.float16)

    def gather(self, x, idx):
        return x[torch.as_tensor(idx)]

    def experts(self, xe, problems, mode):
        a = xe.numpy().view(np.float16)
        if a.shape[0] == 0:
            return xe.clone()
        kw = dict(E=self.el, bias=None)
        if self.bits == 16:
            h, _ = self.o.grouped_gemm(a, problems, bits=16, w16=self.w["w1"], E=self.el,
                                       n=self.lw.f, bias=self.b1, relu=True)
            y, _ = self.o.grouped_gemm(h, problems, bits=16, w16=self.w["w2"], E=self.el,
                                       n=self.d, bias=self.b2, relu=False)
        else:
            h, _ = self.o.grouped_gemm(a, problems, bits=self.bits, packed=self.w["q1"],
                                       scales=self.w["s1"], E=self.el, n=self.lw.f, bias=self.b1,
                                       relu=True)
            y, _ = self.o.grouped_gemm(h, problems, bits=self.bits, packed=self.w["q2"],
                                       scales=self.w["s2"], E=self.el, n=self.d, bias=self.b2,
                                       relu=False)
        del kw
        return _t(y)

    def combine(self, x, fin, k, y_sorted):
        x = x.numpy().view(np.float16)
        out = x.copy()
        for r in range(x.shape[0]):
            if self.fin[r]:
                continue
            acc = x[r]
            for s in range(k):
                prod = (self.y[self.inv[r * k + s]].astype(np.float64) *
                        np.float64(self.scale[r, s])).astype(np.float16)
                acc = (acc.astype(np.float64) + prod.astype(np.float64)).astype(np.float16)
            out[r] = acc
        return _t(out)

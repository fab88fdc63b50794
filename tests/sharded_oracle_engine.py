"""TEST INFRASTRUCTURE: an fp64 CPU engine with the DeviceEngine interface of paper_2406_04984_b200.sharded, built
on the oracle (oracle/meft_oracle.c). It lets tests/test_sharded.py run the expert-sharded orchestration with
world_size 2 over gloo on CPU and compare it with the unsharded reference computation. Approximate scores are the
exact fp64 scores rounded to fp32, so the certified classification has ambiguous candidates to exchange."""
import numpy as np
import torch

from oracle import oracle as O
from paper_2406_04984_b200.sharded import TorchGlue, cert_bound_coeff


class OracleEngine(TorchGlue):
    def __init__(self, w_a, w_b, w_g, rank, world):
        d, M = w_a.shape
        self.d, self.M, self.N = d, M, w_g.shape[0]
        self.M_loc, self.N_loc = M // world, self.N // world
        self.E = M // self.N
        lo, hi = rank * self.M_loc, (rank + 1) * self.M_loc
        self.w_g = np.ascontiguousarray(w_g)
        self.store = O.OracleStore(w_a[:, lo:hi], w_b[lo:hi])  # the local shard, reference layouts

    # ---- selection pieces
    def route(self, h, kk):
        h = h.numpy()
        tau = [O.select_experts(O.route_scores(h[t], self.w_g), kk) for t in range(h.shape[0])]
        return torch.tensor(np.array(tau), dtype=torch.int32)

    def row_stats(self, rows):
        n = np.linalg.norm(rows.numpy().astype(np.float64), axis=1) * (1 + 1e-6)
        return torch.tensor(n.astype(np.float32)), torch.zeros(rows.shape[0], dtype=torch.int32)

    def key_stats(self):
        n = np.linalg.norm(self.store.w_a, axis=0) * (1 + 1e-6)
        return torch.tensor(n.astype(np.float32)), torch.zeros(self.M_loc, dtype=torch.int32)

    def _dot(self, row, key_local):
        return O.lib().or_dot(O._ptr(np.ascontiguousarray(row)), O._ptr(np.ascontiguousarray(self.store.w_a[:, key_local])),
                              O._I64(self.d))

    def score(self, rows, expert_local):
        rows = rows.numpy()
        out = np.empty((rows.shape[0], self.E), np.float32)
        for r in range(rows.shape[0]):
            e = int(expert_local[r])
            for j in range(self.E):
                out[r, j] = np.float32(self._dot(rows[r], e * self.E + j))
        return torch.tensor(out)

    def exact(self, rows, pair_row, pair_key):
        rows = rows.numpy()
        return torch.tensor([self._dot(rows[int(r)], int(k)) for r, k in zip(pair_row, pair_key)], dtype=torch.float64)

    def classify(self, cand, tau, hn, kn, take, d):
        """numpy restatement of k_topk_classify (select_tc.cuh)."""
        cand, tau, hn, kn = cand.numpy(), tau.numpy(), hn.numpy(), kn.numpy()
        T, C = cand.shape
        kk = tau.shape[1]
        E = C // kk
        cb = cert_bound_coeff(d)
        sure = np.zeros((T, take), np.int32)
        amb = np.zeros((T, C), np.int32)
        n_sure = np.zeros(T, np.int32)
        n_amb = np.zeros(T, np.int32)
        for t in range(T):
            g = np.array([tau[t, i // E] * E + i % E for i in range(C)])
            s = cand[t].astype(np.float64)
            order = sorted(range(C), key=lambda i: (-cand[t, i], i))
            top = np.zeros(C, bool)
            top[order[:take]] = True
            e = cb * float(hn[t]) * kn[g].astype(np.float64)
            lin = np.min((s - e)[top])
            uout = np.max((s + e)[~top]) if (~top).any() else -np.inf
            a = (top & (s - e <= uout)) | (~top & (s + e >= lin))
            su = top & ~a
            n_sure[t], n_amb[t] = su.sum(), a.sum()
            sure[t, :su.sum()] = g[su]
            amb[t, :a.sum()] = g[a]
        return torch.tensor(sure), torch.tensor(n_sure), torch.tensor(amb), torch.tensor(n_amb)

    def finalize(self, sure, n_sure, amb, n_amb, x, take, M):
        T = sure.shape[0]
        per = np.zeros((T, take), np.int32)
        flags = torch.zeros(M, dtype=torch.uint8)
        for t in range(T):
            ns, na = int(n_sure[t]), int(n_amb[t])
            cand = sorted(range(na), key=lambda a: (-float(x[t, a]), int(amb[t, a])))[: take - ns]
            chosen = sorted([int(v) for v in sure[t, :ns]] + [int(amb[t, a]) for a in cand])
            per[t] = chosen
            flags[chosen] = 1
        return torch.tensor(per), flags

    # ---- local FFN + scatter + Adam
    def ffn_local(self, h_all, g_all, S_local, lr):
        h, g = h_all.numpy().astype(np.float64), g_all.numpy().astype(np.float64)
        S = S_local.numpy().astype(np.int64)
        wak, wbk = O.gather_adapter(self.store.w_a, self.store.w_b, S)
        out, z, _ = O.ffn_forward(h, wak, wbk)
        gwa, gwb, gh = O.ffn_backward(g, h, z, None, wak, wbk)
        if len(S):
            self.store.scatter_grads(S, gwa, gwb)
            self.store.sparse_adam(lr)
        return torch.tensor(out), torch.tensor(gh)

"""One Silenzio training step (Alg. 6) on encrypted data.

SURVEY.md §8(f) NEXT #1. A host-side sequence of C-ABI gadget calls (every
arithmetic step is a libsilenzio kernel launch: Matmul^RNS, RNS2MRNS,
sign / abs, bit lengths + block max, the 8-bit digit combine, IntCELossDeriv,
and the training gadgets of csrc/gadgets_train.cu); this module only orders
the calls and reshapes ciphertext arrays. There is no CPU fallback: without
the CUDA library every call raises.

Widths and readings (R23-R26): parameter set A (4-bit messages +
padding, Delta = 2^59) for every LUT except the 8-bit MRNS digit combine of
Shift2MSBs+- (set B); alpha = beta = Gamma = 4, ReLU cap x = 7, weights clipped
to [-8, 7]; getRNSBase over {5, 7, 9, 11, 13} + 16. New 4-bit gadgets
(C ABI, csrc/gadgets_train.cu):
  * channel16: the m = 16 residue Matmul^RNS emits at 2^60 -> Delta (2 PBS),
  * sign3: Sign^RNS_(-1,0,1): top MRNS digit >= 8 and the zero
    test (sum of [digit != 0] over the digits) packed into one PBS,
  * relu_cap, relu_mask (ReLU_x and its derivative times an error sign),
  * update: clip(W - G) for G in {-1, 0, 1} as two bit x 4-bit products
    (toolbox T4) plus a refreshing identity PBS.
The cleartext result every step must decrypt to is oracle.gadgets.train_step
(tests/test_gpu_training.py)."""
import math

import numpy as np
import torch

from . import silenzio as sz
from . import workload as wl

W_BITS = 4           # RNS modulus bit width w of Shift2MSBs
BASES4 = [(13, 16), (11, 13, 16), (9, 11, 13, 16), (7, 9, 11, 13, 16), (5, 7, 9, 11, 13, 16)]


def get_rns_base(max_abs: int):
    """getRNSBase (R24): smallest base with M > 2 max_abs + 1."""
    for base in BASES4:
        if math.prod(base) > 2 * max_abs + 1:
            return list(base)
    raise ValueError("no 4-bit RNS base covers the range")


class Context:
    """Keys of both parameter sets and the cross-parameter keyswitching keys."""

    def __init__(self, PA, PB, ka, kb, ksk_ab, pab, ksk_ba, pba, device):
        self.PA, self.PB, self.ka, self.kb = PA, PB, ka, kb
        self.ksk_ab, self.pab, self.ksk_ba, self.pba = ksk_ab, pab, ksk_ba, pba
        self.dev = device
        self.dim = PA.k * PA.N

    # ------------------------------------------------------------- helpers
    def decrypt(self, ct, signed_mod: int = 32):
        """Test/diagnostic helper: decode every row (set-A big key)."""
        ph = wl.to_host_u64(sz.lwe_phase_batch(ct.reshape(-1, self.dim + 1).contiguous(), self.ka["big_key"]))
        v = wl.decode(ph, 4)
        return np.where(2 * v >= signed_mod, v - signed_mod, v)

    # ------------------------------------------------------------- gadgets
    def matmul(self, X, W, base, stream=None):
        """Matmul^RNS (Alg. 2) -> residues [k][a][c] all at Delta (channel16 applied).
        The RNS channels are independent: each modulus runs as its own driver
        call on its own stream, concurrently (a small matmul is a chain of
        latency-bound PBS launches, so the channels overlap instead of queueing)."""
        X, W = X.contiguous(), W.contiguous()

        def one(m):
            def f(st):
                r = sz.rns_matmul(X, W, [m], self.ka["fbsk"], self.ka["ksk"], self.PA, stream=st)[0]
                if m == 16:
                    r = self.channel16(r, st).reshape(r.shape)
                return r
            return f
        if stream is not None:
            with torch.cuda.stream(stream):
                chans = self._par(*[one(m) for m in base])
        else:
            chans = self._par(*[one(m) for m in base])
        return torch.stack(chans)

    def channel16(self, z, stream=None):
        """r at 2^60 (the native mod-16 channel) -> r at Delta (silenzio_channel16)."""
        return sz.channel16(z, self.ka["fbsk"], self.ka["ksk"], self.PA, stream=stream)

    def shift2msbs(self, res, base, times=None):
        """Shift2MSBs+- (Alg. 4) to Gamma = 4: residues [k][count] -> [count] in [-7, 7]
        (silenzio_shift2msbs_pm: the digits-of-x and |x| chains run concurrently)."""
        Y, _ = sz.shift2msbs_pm(res, base, W_BITS, 3, self.ka, self.PA, self.kb, self.PB,
                                self.ksk_ab, self.pab, self.ksk_ba, self.pba)
        self._tick(times, "shift2msbs")
        return Y

    def sign3(self, res, base, stream=None):
        """Sign^RNS_(-1,0,1): [count] in {-1, 0, 1} at Delta (silenzio_rns_sign3)."""
        return sz.rns_sign3(res, base, self.ka["fbsk"], self.ka["ksk"], self.PA, stream=stream)

    def relu_cap(self, S, cap: int):
        return sz.relu_cap(S, cap, self.ka["fbsk"], self.ka["ksk"], self.PA)

    def relu_mask(self, E, S, cap: int, stream=None):
        """E in {-1, 0, 1} times the ReLU_x derivative [0 < S < cap] (R25)."""
        return sz.relu_mask(E, S, cap, self.ka["fbsk"], self.ka["ksk"], self.PA, stream=stream)

    def update(self, W, G, wmin: int = -8, wmax: int = 7, stream=None):
        """clip(W - G) for G in {-1, 0, 1} (silenzio_weight_update)."""
        return sz.weight_update(W, G, wmin, wmax, self.ka["fbsk"], self.ka["ksk"], self.PA, stream=stream)

    def _spawn(self, fn):
        """Start fn(stream) in a background host thread on a new stream ordered
        after the current stream's work; returns a handle for _join."""
        import concurrent.futures as cf
        cur = torch.cuda.current_stream(self.dev)
        st = torch.cuda.Stream(device=self.dev)
        st.wait_stream(cur)
        ex = cf.ThreadPoolExecutor(1)

        def run():
            with torch.cuda.stream(st):
                return fn(st)
        return ex, ex.submit(run), st

    def _join(self, job):
        ex, fut, st = job
        out = fut.result()
        ex.shutdown()
        cur = torch.cuda.current_stream(self.dev)
        cur.wait_stream(st)
        for t in (out if isinstance(out, (tuple, list)) else (out,)):
            if isinstance(t, torch.Tensor):
                t.record_stream(cur)
        return out

    def _par(self, *fns):
        """Run independent gadget chains concurrently: each on its own CUDA stream
        (ordered after the current stream's work) in its own host thread (the
        drivers block on their stream); the current stream then waits for all."""
        import concurrent.futures as cf
        cur = torch.cuda.current_stream(self.dev)
        streams = [torch.cuda.Stream(device=self.dev) for _ in fns]
        for st in streams:
            st.wait_stream(cur)

        def run(f, st):
            with torch.cuda.stream(st):
                return f(st)
        with cf.ThreadPoolExecutor(len(fns)) as ex:
            outs = [f.result() for f in [ex.submit(run, f, st) for f, st in zip(fns, streams)]]
        for st in streams:
            cur.wait_stream(st)
        for o in outs:
            for t in (o if isinstance(o, (tuple, list)) else (o,)):
                if isinstance(t, torch.Tensor):
                    t.record_stream(cur)
        return outs

    # ------------------------------------------------------- one training step
    def _tick(self, times, name):
        if times is not None:
            import time
            torch.cuda.synchronize()
            now = time.perf_counter()
            times[name] = times.get(name, 0.0) + now - times["_t"]
            times["_t"] = now

    def train_step(self, A0, Y, Ws, cap: int = 7, keep=False):
        """A0 [a][b_1], Y [a][c_L] one-hot bits, Ws[l] [c_l][b_l] (ciphertexts
        [..][dim+1] on the device) -> new weights (and intermediates if keep,
        including a per-stage wall-time breakdown)."""
        import time
        L = len(Ws)
        a = A0.shape[0]
        acts, pre, inter = [A0], [], {"pre": [], "acts": [], "errs": [], "grads": []}
        times = {"_t": time.perf_counter()} if keep else None
        tick = lambda name: self._tick(times, name)  # noqa: E731
        for l in range(L):
            W = Ws[l]
            c_l, b_l = W.shape[0], W.shape[1]
            base = get_rns_base(b_l * 64)
            res = self.matmul(acts[-1], W.transpose(0, 1), base)          # [k][a][c_l]
            tick("forward matmul")
            S = self.shift2msbs(res.reshape(len(base), a * c_l, -1), base, times).reshape(a, c_l, -1)
            pre.append(S)
            acts.append(self.relu_cap(S, cap).reshape(a, c_l, -1) if l < L - 1 else S)
            tick("relu")
        E = sz.int_ce_grad(acts[-1].contiguous(), Y.contiguous(), self.ka["fbsk"], self.ka["ksk"], self.PA)
        tick("ce grad")
        inter["errs"].append(E)
        newW = [None] * L
        pending = []
        for l in range(L - 1, -1, -1):
            W = Ws[l]
            c_l, b_l = W.shape[0], W.shape[1]
            gbase = get_rns_base(a * 8)
            Ecur = E

            # gradient branch (G_l, then the weight update) and error branch
            # (E_{l-1}) only read E, W_l and the activations: run them concurrently
            def grad_branch(st, W=W, c_l=c_l, b_l=b_l, l=l, Ecur=Ecur):
                Gm = self.matmul(Ecur.transpose(0, 1), acts[l], gbase, st)
                G = self.sign3(Gm.reshape(len(gbase), c_l * b_l, -1), gbase, st).reshape(c_l, b_l, -1)
                nw = self.update(W.reshape(c_l * b_l, -1), G.reshape(c_l * b_l, -1), stream=st)
                return G, nw.reshape(c_l, b_l, -1)

            def err_branch(st, W=W, c_l=c_l, b_l=b_l, l=l, Ecur=Ecur):
                ebase = get_rns_base(c_l * 8)
                Em = self.matmul(Ecur, W, ebase, st)
                En = self.sign3(Em.reshape(len(ebase), a * b_l, -1), ebase, st)
                return self.relu_mask(En, pre[l - 1].reshape(a * b_l, -1), cap, st).reshape(a, b_l, -1)

            # the gradient branch of layer l is needed only at the end: it runs
            # in the background while the error propagates to the layers below
            pending.append((l, self._spawn(grad_branch)))
            if l > 0:
                E = err_branch(None)
                inter["errs"].append(E)
        grads = [None] * L
        for l, job in pending:
            grads[l], newW[l] = self._join(job)
        inter["grads"] = grads
        tick("backward (gradient | error branches) + update")
        inter["pre"], inter["acts"] = pre, acts
        if times is not None:
            times.pop("_t")
            inter["times"] = times
        return (newW, inter) if keep else newW


def make_context(PA, PB, seed: int, device, ks_ab=(4, 5), ks_ba=(10, 4)):
    """Keys from the seeded draws of synth/ (set A, set B, cross KSKs, R8)."""
    from synth import cross_ksk_randomness, key_randomness
    ra, rb = key_randomness(PA, seed), key_randomness(PB, seed + 1)
    ka, kb = wl.device_keys(PA, ra, device), wl.device_keys(PB, rb, device)
    rab = cross_ksk_randomness(PA.big_dim, ks_ab[1], PB.n, PB.lwe_sigma_log2, seed, 1)
    rba = cross_ksk_randomness(PB.big_dim, ks_ba[1], PA.big_dim, PA.glwe_sigma_log2, seed, 2)
    ksk_ab = sz.ksk_generate(ka["big_key"], kb["lwe_key"], wl.to_dev(rab["ksk_mask"], device),
                             wl.to_dev(rab["ksk_noise"], device), *ks_ab)
    ksk_ba = sz.ksk_generate(kb["big_key"], ka["big_key"], wl.to_dev(rba["ksk_mask"], device),
                             wl.to_dev(rba["ksk_noise"], device), *ks_ba)
    pab = sz.ks_params(PA.big_dim, PB.n, *ks_ab, like=PB)
    pba = sz.ks_params(PB.big_dim, PA.big_dim, *ks_ba, like=PB)
    return Context(PA, PB, ka, kb, ksk_ab, pab, ksk_ba, pba, device)

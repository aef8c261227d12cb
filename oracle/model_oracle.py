"""CPU restatement of the reference amplitude evaluation — TEST INFRASTRUCTURE ONLY.

numpy restatement (fp64, vectorised over samples) of ``AnqsModel`` and
``fill_amplitudes`` from /root/reference/proj:

* ``QuditLayout::make``          src/model.cpp:33-45
* parameter block layout         src/model.cpp:65-80 (per qudit: amplitude block, then phase block;
                                 W1 [hidden][n] row-major, b1, W2 [hidden][hidden], b2, W3 [2^k][hidden], b3)
* ``QuditInfo``                  src/model.cpp:82-93
* ``allowed_values``             src/model.cpp:129-151
* ``encode_prefix``              src/model.cpp:153-158 (+/-1 on the prefix bits, 0 elsewhere)
* ``mlp_forward``                src/model.cpp:160-175 (tanh, residual h1 into the 2nd pre-activation)
* ``conditional``                src/model.cpp:203-252 (mean shift, log-softmax of 2*amp over allowed values)
* ``in_sector`` / ``log_psi``    src/model.cpp:254-271
* ``fill_amplitudes``            src/sampler.cpp:104-120
* ``Philox4x32::block``          src/rng.cpp:15-44 (10 rounds, Weyl key bumps)
* ``CounterRng::gumbel``         include/qvmc/rng.hpp:38-63 (bits64 -> 53-bit uniform, clamp, -log(-log u))
* ``condition_max``              src/sampler.cpp:15-23
* ``sample_without_replacement`` src/sampler.cpp:37-102 (ancestral Gumbel top-K beam, ChildLess order)
* ``grad_log_psi`` / ``mlp_backward`` src/model.cpp:177-325, ``energy_gradient`` src/energy.cpp:93-107
* ``top_probability_indices``, ``build_sr_context``, ``sr_direction`` src/sr.cpp:15-95 (numpy eigh; sr.cpp
  needs Eigen's eigensolver and is not compiled here: pinned to the dense regularised solve, the reference's
  own acceptance check, checks.cpp "SR solve", and its tests in test_energy_sr.cpp)

It is pinned against the reference itself (``oracle/_ref``, model.cpp and
sampler.cpp compiled with the Eigen shim) by tests/test_model.py. Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU legs may import it.
"""
from __future__ import annotations

import numpy as np


def layout(n_qubits: int, bits_per_qudit: int):
    """QuditLayout::make (model.cpp:33-45): (offsets, sizes)."""
    if not 1 <= n_qubits <= 256:
        raise ValueError("QuditLayout: qubit count out of range")
    if not 1 <= bits_per_qudit <= 8:
        raise ValueError("QuditLayout: bits_per_qudit must be in [1, 8]")
    offs = list(range(0, n_qubits, bits_per_qudit))
    return offs, [min(bits_per_qudit, n_qubits - o) for o in offs]


class ModelOracle:
    def __init__(self, n_qubits, bits_per_qudit, n_electrons, spin_constraint, hidden, params):
        self.n, self.hidden = n_qubits, hidden
        self.n_e, self.spin = n_electrons, bool(spin_constraint)
        self.n_up = n_electrons // 2 if self.spin else 0
        self.offsets, self.sizes = layout(n_qubits, bits_per_qudit)
        self.params = np.asarray(params, dtype=np.float64)
        self.blocks = []  # per qudit: (amp, phase), each a dict of views
        cur = 0
        for o, k in zip(self.offsets, self.sizes):
            pair = []
            for _ in range(2):  # model.cpp:65-80
                b = {}
                for name, shape in (("W1", (hidden, n_qubits)), ("b1", (hidden,)), ("W2", (hidden, hidden)),
                                    ("b2", (hidden,)), ("W3", (1 << k, hidden)), ("b3", (1 << k,))):
                    size = int(np.prod(shape))
                    b[name] = self.params[cur:cur + size].reshape(shape)
                    cur += size
                pair.append(b)
            self.blocks.append(pair)
        self.n_params = cur
        if self.params.size != cur:
            raise ValueError("params size mismatch")

    def _info(self, j):  # model.cpp:82-93
        o, k = self.offsets[j], self.sizes[j]
        rem_after = self.n - o - k
        rem_up_after = sum(1 for i in range(o + k, self.n) if i % 2 == 0)
        up_value_mask = 0
        for t in range(k):
            if (o + t) % 2 == 0:
                up_value_mask |= 1 << (k - 1 - t)
        return rem_after, rem_up_after, up_value_mask

    def allowed(self, j, prefix_weight, prefix_up):
        """allowed_values (model.cpp:129-151), vectorised: bool [N][2^k]."""
        k = self.sizes[j]
        rem_after, rem_up_after, upm = self._info(j)
        v = np.arange(1 << k)
        pv = np.array([bin(a).count("1") for a in v])
        pu = np.array([bin(a & upm).count("1") for a in v])
        w = prefix_weight[:, None] + pv[None, :]
        ok = (w <= self.n_e) & (w + rem_after >= self.n_e)
        if self.spin:
            wu = prefix_up[:, None] + pu[None, :]
            wd = w - wu
            n_down = self.n_e - self.n_up
            rem_down = rem_after - rem_up_after
            ok &= (wu <= self.n_up) & (wu + rem_up_after >= self.n_up) & (wd <= n_down) & (wd + rem_down >= n_down)
        return ok

    @staticmethod
    def _mlp(b, e):  # model.cpp:160-175
        h1 = np.tanh(e @ b["W1"].T + b["b1"])
        h2 = np.tanh(h1 @ b["W2"].T + b["b2"] + h1)
        return h2 @ b["W3"].T + b["b3"]

    def log_psi(self, keys):
        """log_psi (model.cpp:262-271) for keys uint64 [N][W]: (log_amp, phase)."""
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        N = keys.shape[0]
        bits = np.unpackbits(keys.view(np.uint8).reshape(N, -1), axis=1, bitorder="little")[:, :self.n].astype(np.int64)
        la = np.zeros(N)
        ph = np.zeros(N)
        pop = bits.sum(1)
        ins = pop == self.n_e  # in_sector (model.cpp:254-259)
        if self.spin:
            ins &= bits[:, 0::2].sum(1) == self.n_up
        for j, (o, k) in enumerate(zip(self.offsets, self.sizes)):
            e = np.zeros((N, self.n))
            e[:, :o] = np.where(bits[:, :o] == 1, 1.0, -1.0)  # encode_prefix
            amp = self._mlp(self.blocks[j][0], e)
            phase = self._mlp(self.blocks[j][1], e)
            amp = amp - amp.mean(axis=1, keepdims=True)  # global activation
            ok = self.allowed(j, bits[:, :o].sum(1), bits[:, 0:o:2].sum(1))
            two = np.where(ok, 2.0 * amp, -np.inf)
            mx = two.max(axis=1)
            with np.errstate(invalid="ignore", over="ignore"):
                lse = mx + np.log(np.where(ok, np.exp(two - mx[:, None]), 0.0).sum(1))
            v = np.zeros(N, dtype=np.int64)
            for t in range(k):  # extract_bits (basis_vector.cpp:40-45): qubit o+t -> bit k-1-t
                v |= bits[:, o + t] << (k - 1 - t)
            rows = np.arange(N)
            la += 0.5 * (2.0 * amp[rows, v] - lse)
            ph += phase[rows, v]
        la = np.where(ins, la, -np.inf)
        ph = np.where(ins, ph, 0.0)
        return la, ph

    def fill_amplitudes(self, keys, log_probs):
        """fill_amplitudes (sampler.cpp:104-120): (log_amps, phases, norm, log_norm)."""
        la, ph = self.log_psi(keys)
        lp = np.asarray(log_probs, dtype=np.float64)
        mx = lp.max()
        log_norm = mx + np.log(np.exp(lp - mx).sum())
        return la, ph, float(np.exp(log_norm)), float(log_norm)


# ---------------------------------------------------------------- sampler restatement

_M0, _M1, _W0, _W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
_U32 = 0xFFFFFFFF


def philox4x32(counter, key):
    """Philox4x32::block (rng.cpp:15-44): 10 rounds, key bumped by the Weyl constants."""
    c = list(counter)
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + _W0) & _U32
            k1 = (k1 + _W1) & _U32
        p0 = _M0 * c[0]
        p1 = _M1 * c[2]
        hi0, lo0, hi1, lo1 = p0 >> 32, p0 & _U32, p1 >> 32, p1 & _U32
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
    return c


def counter_gumbel(seed, stream, c0, c1, c2, c3):
    """CounterRng(seed, stream).gumbel(c0..c3) (rng.hpp:38-63)."""
    key = (seed & _U32, ((seed >> 32) & _U32) ^ stream)
    out = philox4x32((c0, c1, c2, c3), key)
    b = (out[1] << 32) | out[0]
    u = (b >> 11) * 2.0 ** -53
    u = 1e-300 if u < 1e-300 else (1.0 - 1e-16 if u > 1.0 - 1e-16 else u)
    return -np.log(-np.log(u))


def condition_max(parent, z, child):
    """condition_max (sampler.cpp:15-23)."""
    if child == z:
        return parent
    m = max(-parent, -child)
    v = np.exp(-parent - m) - np.exp(-z - m) + np.exp(-child - m)
    if not v > 0.0:
        return parent
    return min(-(m + np.log(v)), parent)


def _key_tuple(k):
    return tuple(int(w) for w in k)  # BasisVector operator< = std::array words_ order (basis_vector.hpp:109-111)


def _deposit(key, offset, count, value):
    """deposit_bits (basis_vector.cpp:47-50): qubit offset+t <- bit count-1-t of value."""
    out = np.array(key, dtype=np.uint64)
    for t in range(count):
        q = offset + t
        bit = (value >> (count - 1 - t)) & 1
        w, b = q // 64, np.uint64(q % 64)
        if bit:
            out[w] |= np.uint64(1) << b
        else:
            out[w] &= ~(np.uint64(1) << b)
    return out



def conditional_log_probs(model: "ModelOracle", prefixes, j):
    """conditional(prefix, j).log_prob (model.cpp:203-252) for a batch of prefixes: [N][2^k], -inf if disallowed."""
    prefixes = np.ascontiguousarray(prefixes, dtype=np.uint64)
    N = prefixes.shape[0]
    bits = np.unpackbits(prefixes.view(np.uint8).reshape(N, -1), axis=1, bitorder="little")[:, :model.n].astype(np.int64)
    o = model.offsets[j]
    e = np.zeros((N, model.n))
    e[:, :o] = np.where(bits[:, :o] == 1, 1.0, -1.0)
    amp = ModelOracle._mlp(model.blocks[j][0], e)
    amp = amp - amp.mean(axis=1, keepdims=True)
    ok = model.allowed(j, bits[:, :o].sum(1), bits[:, 0:o:2].sum(1))
    if not ok.any(axis=1).all():
        raise RuntimeError("AnqsModel::conditional: unreachable prefix")
    two = np.where(ok, 2.0 * amp, -np.inf)
    mx = two.max(axis=1)
    lse = mx + np.log(np.where(ok, np.exp(two - mx[:, None]), 0.0).sum(1))
    return np.where(ok, two - lse[:, None], -np.inf)


def sample_without_replacement(model: "ModelOracle", k_samples, seed, stream=0, iteration=0):
    """sample_without_replacement (sampler.cpp:37-102): (keys [n][W], log_probs [n]) in ChildLess order."""
    if k_samples < 1:
        raise ValueError("sample_without_replacement: K must be >= 1")
    W = (model.n + 63) // 64
    beam = [(np.zeros(W, dtype=np.uint64), 0.0, 0.0)]  # (prefix, log_prob, perturbed)
    for level, (off, k) in enumerate(zip(model.offsets, model.sizes)):
        cond = conditional_log_probs(model, np.stack([b[0] for b in beam]), level)
        children = []
        for b, (prefix, lp, pert) in enumerate(beam):
            out = []
            z = -np.inf
            for v in range(1 << k):
                if cond[b, v] == -np.inf:
                    continue
                clp = lp + cond[b, v]
                u = clp + counter_gumbel(seed, stream, iteration, level, b, v)
                z = max(z, u)
                out.append([_deposit(prefix, off, k, v), clp, u])
            for c in out:
                c[2] = condition_max(pert, z, c[2])
            children += out
        if not children:
            raise RuntimeError("sample_without_replacement: empty sector")
        children.sort(key=lambda c: (-c[2], _key_tuple(c[0])))  # ChildLess (sampler.cpp:27-33)
        beam = [tuple(c) for c in children[:k_samples]]
    return np.stack([b[0] for b in beam]), np.array([b[1] for b in beam])


# ---------------------------------------------------------------- gradient restatement

def _mlp_fwd(b, e):
    h1 = np.tanh(e @ b["W1"].T + b["b1"])
    h2 = np.tanh(h1 @ b["W2"].T + b["b2"] + h1)
    return h1, h2, h2 @ b["W3"].T + b["b3"]


def _mlp_bwd(b, e, h1, h2, g):
    """mlp_backward (model.cpp:177-201), rows = samples: per-sample blocks (W1, b1, W2, b2, W3, b3)."""
    gz2 = (g @ b["W3"]) * (1.0 - h2 ** 2)
    gh1 = gz2 @ b["W2"] + gz2
    gz1 = gh1 * (1.0 - h1 ** 2)
    N = e.shape[0]
    return [np.einsum("sh,si->shi", gz1, e).reshape(N, -1), gz1, np.einsum("sh,sk->shk", gz2, h1).reshape(N, -1),
            gz2, np.einsum("sv,sh->svh", g, h2).reshape(N, -1), g]


def grad_log_psi(model: "ModelOracle", keys):
    """batched_grad_log_psi (model.cpp:273-336): complex rows [N][n_params], d log|psi| - i d phase."""
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    N = keys.shape[0]
    bits = np.unpackbits(keys.view(np.uint8).reshape(N, -1), axis=1, bitorder="little")[:, :model.n].astype(np.int64)
    la, _ = model.log_psi(keys)
    if not np.all(np.isfinite(la)):
        raise ValueError("grad_log_psi: state is masked (zero amplitude)")
    rows = []
    for j, (o, k) in enumerate(zip(model.offsets, model.sizes)):
        e = np.zeros((N, model.n))
        e[:, :o] = np.where(bits[:, :o] == 1, 1.0, -1.0)
        v = np.zeros(N, dtype=np.int64)
        for t in range(k):
            v |= bits[:, o + t] << (k - 1 - t)
        onehot = np.zeros((N, 1 << k))
        onehot[np.arange(N), v] = 1.0
        ab, pb = model.blocks[j]
        h1, h2, out = _mlp_fwd(ab, e)
        out = out - out.mean(axis=1, keepdims=True)
        ok = model.allowed(j, bits[:, :o].sum(1), bits[:, 0:o:2].sum(1))
        two = np.where(ok, 2.0 * out, -np.inf)
        mx = two.max(axis=1, keepdims=True)
        ex = np.where(ok, np.exp(two - mx), 0.0)
        g = onehot - ex / ex.sum(axis=1, keepdims=True)
        g = g - g.mean(axis=1, keepdims=True)
        rows += [blk.astype(np.complex128) for blk in _mlp_bwd(ab, e, h1, h2, g)]
        h1p, h2p, _ = _mlp_fwd(pb, e)
        rows += [-1j * blk for blk in _mlp_bwd(pb, e, h1p, h2p, onehot)]
    return np.concatenate(rows, axis=1)


def energy_gradient(weights, locals_, jacobian):
    """energy_gradient (energy.cpp:93-107): sum_i 2 Re{w_i (E_i - E) row_i}, E = sum_i w_i E_i."""
    w = np.asarray(weights, dtype=np.float64)
    loc = np.asarray(locals_, dtype=np.complex128)
    c = w * (loc - (w * loc).sum())
    return 2.0 * (c.real @ jacobian.real - c.imag @ jacobian.imag)


# ---------------------------------------------------------------- SR restatement

def top_probability_indices(log_probs, n_sr):
    """top_probability_indices (sr.cpp:15-23): stable sort by log p descending."""
    lp = np.asarray(log_probs, dtype=np.float64)
    return np.argsort(-lp, kind="stable")[: min(n_sr, lp.size)]


def build_sr_context(log_probs, locals_, selected, jac_rows, lam=0.0):
    """build_sr_context (sr.cpp:25-72): (stacked [2n][P], f_stacked [2n], lambda)."""
    lp = np.asarray(log_probs, dtype=np.float64)[selected]
    n = len(selected)
    if n < 1:
        raise ValueError("build_sr_context: empty selection")
    w = np.exp(lp - lp.max())
    w /= w.sum()
    row_mean = (w[:, None] * jac_rows).sum(0)
    loc = np.asarray(locals_, dtype=np.complex128)[selected]
    e_mean = (w * loc).sum()
    s = np.sqrt(w)
    centered = (jac_rows - row_mean) * s[:, None]
    stacked = np.concatenate([centered.real, centered.imag])
    f = s * np.conj(loc - e_mean)
    f_stacked = np.concatenate([f.real, f.imag])
    lam = lam if lam > 0.0 else 1e-4 * (1.0 + (stacked ** 2).sum() / n)
    return stacked, f_stacked, lam


def sr_direction(stacked, lam, grad):
    """sr_direction (sr.cpp:74-95): push-through identity with the Gram eigensystem."""
    gram = stacked @ stacked.T + lam * np.eye(stacked.shape[0])
    ev, V = np.linalg.eigh(gram)
    lo, hi = ev.min(), ev.max()
    if not lo > 0.0 or hi / lo > 1e14:
        raise RuntimeError(f"sr_direction: ill-conditioned system, cond ~ {hi / max(lo, 1e-300)}")
    t = stacked @ grad
    s = V @ ((V.T @ t) / ev)
    return (grad - stacked.T @ s) / lam

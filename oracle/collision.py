"""The fast-spectral collision operator, two evaluators of one definition (oracle; tests only).

Definition (readings #9/#10): with F_l = n^{-1} sum_j f_j e^{-2 pi i l.j/N}
(the DFT of the node values, P:386 up to the node phase, which cancels in index space),

    Qhat_k = sum_{l} beta(l, k (-) l) F_l F_{k (-) l},
    beta(l, m) = sum_p w_p alpha_p(l) alpha'_p(m) - D(m)

where k (-) l wraps each component into [-N/2, N/2) -- the circular convolution that
pointwise products of N-point inverse DFTs compute (reading #9).  Back at the nodes:

    Q_j = s * Re sum_k Qhat_k e^{+2 pi i k.j/N},   s = Btilde kappa^{-(d+gamma)}.

``collide_direct`` evaluates the double sum literally (O(n^2 A)); it is the parity truth.
``collide_fft`` evaluates the same bilinear form by the convolution theorem (P:451,
"A discrete convolutions ... by means of standard FFT technique"):

    Q = s [ sum_p w_p a_p b_p - f c ],  a_p = IDFT(alpha_p F), b_p = IDFT(alpha'_p F),
                                         c = IDFT(D F)

with IDFT(X)_j = sum_k X_k e^{+2 pi i k.j/N}.  It is pinned to ``collide_direct`` (P4).
Both return Q in user units, unprojected, without 1/tau.
"""
import numpy as np


def dft(f):
    """F_l = n^{-1} sum_j f_j e^{-2 pi i l.j/N} (numpy.fft as a library primitive, pin P1)."""
    return np.fft.fftn(f) / f.size


def idft(X):
    """IDFT(X)_j = sum_k X_k e^{+2 pi i k.j/N}."""
    return np.fft.ifftn(X) * X.size


def _wrap_index_matrix(shape):
    """idx[k, l] = flat index of (k - l) mod N per axis, for all flat k, l."""
    n = int(np.prod(shape))
    coords = np.array(np.unravel_index(np.arange(n), shape))  # [d, n]
    diff = (coords[:, :, None] - coords[:, None, :]) % np.array(shape)[:, None, None]
    return np.ravel_multi_index(tuple(diff), shape)


def qhat_direct(f, tab, modes=None):
    """Qhat_k (before the factor s) by the literal double sum, for all k or the flat mode
    indices ``modes``.  Returns (Qhat, Qhat_gain, Qhat_loss)."""
    shape = f.shape
    n = f.size
    F = dft(f).reshape(-1)
    coords = np.array(np.unravel_index(np.arange(n), shape))  # [d, n]
    ks = np.arange(n) if modes is None else np.asarray(modes)
    kc = np.array(np.unravel_index(ks, shape))  # [d, K]
    diff = (kc[:, :, None] - coords[:, None, :]) % np.array(shape)[:, None, None]
    m_idx = np.ravel_multi_index(tuple(diff), shape)  # [K, n]: m = k (-) l
    Fm = F[m_idx]                                     # F_{k-l}
    gain = np.zeros(len(ks), dtype=np.complex128)
    for p in range(tab.A):
        al = tab.alpha[p].reshape(-1)
        alp = tab.alphap[p].reshape(-1)
        gain += tab.w[p] * np.sum((al * F)[None, :] * alp[m_idx] * Fm, axis=1)
    D = tab.D.reshape(-1)
    loss = np.sum(F[None, :] * D[m_idx] * Fm, axis=1)
    return gain - loss, gain, loss


def collide_direct(f, tab, return_parts=False):
    """Q at the nodes from the literal O(n^2 A) bilinear form."""
    Qh, Qg, Ql = qhat_direct(f, tab)
    shape = f.shape
    Q = idft(Qh.reshape(shape))
    assert np.max(np.abs(Q.imag)) <= 1e-13 * max(np.max(np.abs(idft(Ql.reshape(shape)))), 1e-300), \
        "imaginary residue: tables not even (reading #10)"
    Q = tab.scale * Q.real
    if return_parts:
        return Q, tab.scale * idft(Qg.reshape(shape)).real, tab.scale * idft(Ql.reshape(shape)).real
    return Q


def collide_fft(f, tab, return_parts=False):
    """The same bilinear form through the convolution theorem."""
    F = dft(f)
    G = np.zeros(f.shape)
    for p in range(tab.A):
        a = idft(tab.alpha[p] * F).real
        b = idft(tab.alphap[p] * F).real
        G += tab.w[p] * a * b
    c = idft(tab.D * F).real
    gain = tab.scale * G
    loss = tab.scale * f * c
    Q = gain - loss
    if return_parts:
        return Q, gain, loss
    return Q


def collide_fft_batch(fs, tab):
    """collide_fft over a leading batch axis."""
    return np.stack([collide_fft(f, tab) for f in fs])

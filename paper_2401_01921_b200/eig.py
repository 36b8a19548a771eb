"""Device-resident Lanczos for the DMRG effective Hamiltonian.

Same contract as the reference (pkg/src/tnkit/linalg.py:445-562): ``LinOp`` wraps a
Hermitian map of fixed dimension; ``lanczos(op, k, v0, tol, max_iter, seed)`` runs
Lanczos with full reorthogonalisation, declares convergence when every target
Ritz value has residual ``|op(v) - theta v| <= tol * max(1, |theta|)``, restarts on
breakdown with a fresh orthogonal random vector, and raises ``ConvergenceError``
carrying the best estimate. Here the Krylov basis and every vector operation live
in HBM; the matvec is an engine call (e.g. a compiled L.A.W.R Network replayed as
a CUDA graph, ``NetworkMatvec``); only the alpha/beta scalars and the small
tridiagonal problem cross to the host.
"""
import numpy as np
import scipy.linalg
import torch

from . import dense


class ConvergenceError(RuntimeError):
    def __init__(self, message, eigenvalues=None, eigenvectors=None):
        super().__init__(message)
        self.eigenvalues = eigenvalues
        self.eigenvectors = eigenvectors


class LinOp:
    """A Hermitian linear map on device vectors (1-D torch tensors)."""

    def __init__(self, dim, matvec=None, dtype=np.float64, hermitian=True):
        if dim < 1:
            raise ValueError(f"operator dimension must be >= 1, got {dim}")
        self.dim = int(dim)
        self.dtype = np.dtype(dtype)
        self.hermitian = bool(hermitian)
        self._matvec = matvec

    def matvec(self, v):
        if self._matvec is None:
            raise NotImplementedError("override matvec or pass a callable")
        return self._matvec(v)

    def __call__(self, v):
        out = self.matvec(v)
        if tuple(out.shape) != (self.dim,):
            raise ValueError(f"operator returned shape {tuple(out.shape)}, expected ({self.dim},)")
        return out


class NetworkMatvec(LinOp):
    """``op(v) = Network(...).launch()`` with slot `slot` bound to `v` (reshaped like
    the captured tensor): the Lanczos inner loop of DMRG (tnkit dmrg.py:271-286)
    as one graph replay per iteration on device buffers."""

    def __init__(self, compiled, slot, out_perm=None):
        self.compiled = compiled
        self.slot = slot
        src = compiled.input(slot)
        if src.is_sym:
            raise TypeError("NetworkMatvec needs a dense slot")
        self._in = src.get_block_()
        self._out_perm = out_perm
        super().__init__(self._in.size, dtype=src.dtype)

    def matvec(self, v):
        self._in.view().copy_(v.view(self._in.shape))
        out = self.compiled.launch()
        blk = out.get_block_()
        if self._out_perm is not None:
            blk = blk.permute(*self._out_perm)
        return blk.contiguous().storage().clone()


def _tt(np_dtype):
    return dense._TORCH[np.dtype(np_dtype)]


def lanczos(op, k=1, v0=None, tol=1e-12, max_iter=None, seed=None):
    """Lowest ``k`` eigenpairs; returns (values ascending (numpy), vectors as columns (device))."""
    if not isinstance(op, LinOp):
        raise TypeError("lanczos expects a LinOp")
    if not op.hermitian:
        raise ValueError("lanczos requires an operator declared Hermitian")
    n = op.dim
    if not 1 <= k <= n:
        raise ValueError(f"need 1 <= k <= dim, got k={k}, dim={n}")
    if max_iter is None:
        max_iter = min(10 * n, 10000)
    dev = dense.device()
    tdt = _tt(op.dtype)
    cplx = np.issubdtype(op.dtype, np.complexfloating)
    rng = np.random.default_rng(seed if seed is not None else 20240527)

    def random_start():
        v = rng.standard_normal(n)
        if cplx:
            v = v + 1j * rng.standard_normal(n)
        return torch.from_numpy(np.asarray(v, dtype=op.dtype)).to(dev)

    if v0 is None:
        q = random_start()
    else:
        q = (v0 if isinstance(v0, torch.Tensor) else torch.from_numpy(np.asarray(v0, dtype=op.dtype))).to(dev, tdt)
        if tuple(q.shape) != (n,):
            raise ValueError(f"v0 has shape {tuple(q.shape)}, expected ({n},)")
    if float(torch.linalg.vector_norm(q)) == 0.0:
        q = random_start()
    q = q / torch.linalg.vector_norm(q)
    m_max = min(max_iter, n)
    # Krylov basis stored as ROWS (contiguous vectors): the reorthogonalisation is two
    # row-major GEMVs and every basis access is a contiguous vector
    Qt = torch.zeros((m_max + 1, n), dtype=tdt, device=dev)
    Qt[0] = q
    alphas, betas = [], []
    it = 0
    scale = 1.0

    def ritz(count):
        theta, y = scipy.linalg.eigh_tridiagonal(np.asarray(alphas), np.asarray(betas), select="i",
                                                 select_range=(0, count - 1))
        return theta, y

    def vectors(mdim, y):
        return Qt[:mdim].T @ torch.from_numpy(y.astype(op.dtype)).to(dev)

    while True:
        w = op(Qt[it])
        alpha = float(torch.vdot(Qt[it], w).real)
        alphas.append(alpha)
        scale = max(scale, abs(alpha))
        w = w - alpha * Qt[it]
        if it > 0:
            w = w - betas[-1] * Qt[it - 1]
        basis = Qt[:it + 1]
        w = w - basis.T @ (basis.conj() @ w)  # full reorthogonalisation
        beta = float(torch.linalg.vector_norm(w))
        mdim = it + 1
        if mdim >= k:
            theta, y = ritz(k)
            resid = beta * np.abs(y[-1, :])
            if np.all(resid <= tol * np.maximum(1.0, np.abs(theta))) or mdim == n:
                return theta, vectors(mdim, y)
        if mdim >= m_max:
            theta, y = ritz(min(k, mdim))
            raise ConvergenceError(
                f"lanczos did not converge within {max_iter} iterations "
                f"(best residual {float(np.max(beta * np.abs(y[-1, :]))):.3e})",
                eigenvalues=theta, eigenvectors=vectors(mdim, y))
        if beta <= 1e-13 * scale:
            w = random_start()
            w = w - basis.T @ (basis.conj() @ w)
            nw = float(torch.linalg.vector_norm(w))
            if nw < 1e-12:
                theta, y = ritz(min(k, mdim))
                return theta, vectors(mdim, y)
            betas.append(0.0)
            Qt[mdim] = w / nw
        else:
            betas.append(beta)
            Qt[mdim] = w / beta
        it += 1

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


class _DeviceSteps:
    """Krylov basis (rows of Qt), alpha / beta per iteration and the step workspace in HBM;
    tnb_lanczos_step does the vector work, one small async copy per iteration brings
    (alpha, beta) to pinned host memory."""

    def __init__(self, n, m_max, op_dtype, dev):
        from . import _lib
        self.n = n
        self.code = dense.dtype_code(np.dtype(op_dtype))
        self.Qt = torch.zeros((m_max + 1, n), dtype=_tt(op_dtype), device=dev)
        self.ab = torch.zeros((m_max + 2, 2), dtype=torch.float64, device=dev)
        self.host = torch.zeros((m_max + 2, 2), dtype=torch.float64).pin_memory()
        self.scratch = torch.zeros(2, dtype=torch.float64, device=dev)
        self.work = torch.zeros(_lib.lanczos_work_bytes(m_max + 1, n), dtype=torch.uint8, device=dev)
        self.events = {}
        self.isz = self.Qt.element_size()
        self._lib = _lib

    def step(self, r, w, q_next_row, slot=None):
        """Reorthogonalise w against rows [0, r) of Qt; w / |w| -> Qt[q_next_row]. alpha / beta
        go to ab[slot] (or the scratch pair) and are copied to the host asynchronously."""
        ab = self.ab[slot] if slot is not None else self.scratch
        qn = self.Qt[q_next_row].data_ptr() if q_next_row is not None else None
        self._lib.lanczos_step(self.code, self.Qt.data_ptr(), self.n, r, w.data_ptr(), self.n, qn,
                               ab.data_ptr(), ab.data_ptr() + 8, self.work.data_ptr(), dense.stream_handle())
        if slot is not None:
            self.host[slot].copy_(ab, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self.events[slot] = ev

    def read(self, slot):
        self.events.pop(slot).synchronize()
        a, b = self.host[slot].tolist()
        return a, b

    def read_scratch(self):
        a, b = self.scratch.tolist()  # synchronising (rare: start / restart vectors)
        return a, b

    def vectors(self, mdim, y):
        """Ritz vectors Qt[:mdim]^T y as columns [n, k] (one engine contraction)."""
        from . import _lib
        ydt = np.complex128 if self.Qt.dtype == torch.complex128 else np.float64
        yk = torch.from_numpy(np.ascontiguousarray(y.astype(ydt))).to(self.Qt.device)
        out = torch.empty((self.n, yk.shape[1]), dtype=self.Qt.dtype, device=self.Qt.device)
        _lib.contract_dense(self.Qt.data_ptr(), self.code, (mdim, self.n), (0, 1), yk.data_ptr(), self.code,
                            tuple(yk.shape), (0, 1), [0], [0], out.data_ptr(), _lib.CPLX_4M, dense.stream_handle())
        return out


def lanczos(op, k=1, v0=None, tol=1e-12, max_iter=None, seed=None):
    """Lowest ``k`` eigenpairs; returns (values ascending (numpy), vectors as columns (device)).

    Vector work on the device (tnb_lanczos_step), alpha / beta read back one iteration
    behind: iteration i+1's matvec is enqueued before iteration i's scalars are checked, so
    the host never stalls the GPU. Converging at iteration i returns the state after
    iteration i exactly (the speculative step only wrote basis row i+2)."""
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
        q = q.clone()
    m_max = min(max_iter, n)
    ds = _DeviceSteps(n, m_max, op.dtype, dev)
    ds.step(0, q, 0)  # Qt[0] = q / |q|
    if ds.read_scratch()[1] == 0.0:
        ds.step(0, random_start(), 0)
    alphas, betas = [], []
    scale = 1.0

    def ritz(count):
        return scipy.linalg.eigh_tridiagonal(np.asarray(alphas), np.asarray(betas), select="i",
                                             select_range=(0, count - 1))

    def launch(i):  # matvec on basis row i, then the device step writing basis row i + 1
        w = op(ds.Qt[i])
        ds.step(i + 1, w, i + 1 if i + 1 <= m_max else None, slot=i)

    it = 0
    launch(0)
    while True:
        if it + 1 < m_max:
            launch(it + 1)  # speculative: valid unless iteration `it` breaks down
        alpha, beta = ds.read(it)
        alphas.append(alpha)
        scale = max(scale, abs(alpha))
        mdim = it + 1
        if mdim >= k:
            theta, y = ritz(k)
            resid = beta * np.abs(y[-1, :])
            if np.all(resid <= tol * np.maximum(1.0, np.abs(theta))) or mdim == n:
                return theta, ds.vectors(mdim, y)
        if mdim >= m_max:
            theta, y = ritz(min(k, mdim))
            raise ConvergenceError(
                f"lanczos did not converge within {max_iter} iterations "
                f"(best residual {float(np.max(beta * np.abs(y[-1, :]))):.3e})",
                eigenvalues=theta, eigenvectors=ds.vectors(mdim, y))
        if beta <= 1e-13 * scale:
            # breakdown: restart with a random vector orthogonal to the basis (the speculative
            # iteration it + 1 read a meaningless row; it is redone below)
            if it + 1 < m_max:
                ds.read(it + 1)
            ds.step(mdim, random_start(), mdim)
            if ds.read_scratch()[1] < 1e-12:
                theta, y = ritz(min(k, mdim))
                return theta, ds.vectors(mdim, y)
            betas.append(0.0)
            if it + 1 < m_max:
                launch(it + 1)
        else:
            betas.append(beta)
        it += 1

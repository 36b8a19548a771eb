"""Abelian charge algebra and bonds (host-side integer bookkeeping).

Mirrors the reference's public interface -- ``Symmetry`` (pkg/src/tnkit/
symmetry.py:14-89), the qnum tuple helpers (symmetry.py:101-130) and ``Bond`` /
``BondType`` (bond.py:16-196) -- because sector order and degeneracies define
block shapes and ``Bond.__eq__`` gates contraction (contract.py:84-97). All of
it must agree with the reference bit for bit; it never touches the GPU.
"""
import enum

U1 = "U1"
ZN = "Zn"


class Symmetry:
    """U(1) (unbounded integers under +) or Z_n (integers mod n)."""

    __slots__ = ("kind", "n")

    def __init__(self, kind, n=0):
        if kind == ZN:
            if n < 2:
                raise ValueError(f"Zn requires n >= 2, got n={n}")
            self.n = int(n)
        elif kind == U1:
            self.n = 0
        else:
            raise ValueError(f"unknown symmetry kind: {kind!r}")
        self.kind = kind

    @classmethod
    def u1(cls):
        return cls(U1)

    @classmethod
    def zn(cls, n):
        return cls(ZN, n)

    @property
    def modulus(self):
        """0 for U(1), n for Z_n (the ABI's sym_n code)."""
        return self.n

    def normalize(self, q):
        q = int(q)
        return q % self.n if self.n else q

    def combine(self, q1, q2):
        return (q1 + q2) % self.n if self.n else q1 + q2

    def reverse(self, q):
        return (-q) % self.n if self.n else -q

    @property
    def identity(self):
        return 0

    def __eq__(self, other):
        if not isinstance(other, Symmetry):
            return NotImplemented
        return (self.kind, self.n) == (other.kind, other.n)

    def __hash__(self):
        return hash((self.kind, self.n))

    def __str__(self):
        return f"Z{self.n}" if self.n else "U1"

    def __repr__(self):
        return f"Symmetry.zn({self.n})" if self.n else "Symmetry.u1()"


def symmetry_from_str(tag):
    if tag == "U1":
        return Symmetry.u1()
    if tag[:1] == "Z" and tag[1:].isdigit():
        return Symmetry.zn(int(tag[1:]))
    raise ValueError(f"unknown symmetry tag: {tag!r}")


def as_qnum(q, syms):
    """int or sequence -> normalized tuple with one component per symmetry."""
    comps = (q,) if isinstance(q, int) else tuple(int(x) for x in q)
    if len(comps) != len(syms):
        raise ValueError(f"quantum number {comps} has {len(comps)} components, expected {len(syms)}")
    return tuple(s.normalize(x) for s, x in zip(syms, comps))


def combine_qnums(qa, qb, syms):
    return tuple(s.combine(x, y) for s, x, y in zip(syms, qa, qb))


def reverse_qnums(q, syms):
    return tuple(s.reverse(x) for s, x in zip(syms, q))


def identity_qnum(syms):
    return tuple(0 for _ in syms)


class BondType(enum.Enum):
    REGULAR = 0
    IN = 1
    OUT = -1

    def __str__(self):
        return self.name


REGULAR = BondType.REGULAR
IN = BondType.IN
OUT = BondType.OUT


class Bond:
    """One tensor index: dimension, direction, ordered (qnum, degeneracy) sectors."""

    __slots__ = ("btype", "dim", "sectors", "syms", "_offsets")

    def __init__(self, dim=None, btype=REGULAR, sectors=None, syms=None):
        if not isinstance(btype, BondType):
            raise TypeError("btype must be a BondType")
        self.btype = btype
        self._offsets = None
        if sectors is None:
            if dim is None or int(dim) < 1:
                raise ValueError(f"bond dimension must be >= 1, got {dim}")
            if syms:
                raise ValueError("a symmetry list requires sectors")
            self.dim, self.sectors, self.syms = int(dim), (), ()
            return
        if dim is not None:
            raise ValueError("pass either dim or sectors, not both")
        if btype == REGULAR:
            raise ValueError("bonds with quantum numbers must be directed")
        if not syms:
            raise ValueError("sectors require a symmetry list")
        if len(sectors) == 0:
            raise ValueError("sector list must not be empty")
        syms = tuple(syms)
        normed, seen = [], set()
        for qn, deg in sectors:
            qn, deg = as_qnum(qn, syms), int(deg)
            if deg < 1:
                raise ValueError(f"degeneracy must be >= 1, got {deg}")
            if qn in seen:
                raise ValueError(f"duplicate quantum number {qn} in bond")
            seen.add(qn)
            normed.append((qn, deg))
        self.sectors = tuple(normed)
        self.syms = syms
        self.dim = sum(d for _, d in normed)

    @property
    def has_qnums(self):
        return len(self.sectors) > 0

    @property
    def nsectors(self):
        return len(self.sectors)

    def qnums(self):
        return tuple(q for q, _ in self.sectors)

    def degeneracies(self):
        return tuple(d for _, d in self.sectors)

    def sector_offsets(self):
        if self._offsets is None:
            acc, offs = 0, []
            for d in self.degeneracies():
                offs.append(acc)
                acc += d
            self._offsets = tuple(offs)
        return self._offsets

    def locate(self, index):
        """flat index -> (sector position, offset inside the sector)"""
        if not 0 <= index < self.dim:
            raise IndexError(f"index {index} out of range for bond of dim {self.dim}")
        for pos, start in enumerate(self.sector_offsets()):
            if index < start + self.sectors[pos][1]:
                return pos, index - start
        raise AssertionError("unreachable")

    def combine(self, other):
        """Tensor product; equal charges grouped in first-appearance order."""
        if isinstance(other, (list, tuple)):
            acc = self
            for b in other:
                acc = acc.combine(b)
            return acc
        if not isinstance(other, Bond):
            raise TypeError("can only combine with another Bond")
        if self.btype != other.btype:
            raise ValueError(f"only bonds with the same direction can be combined "
                             f"({self.btype} vs {other.btype})")
        if self.syms != other.syms:
            raise ValueError("bonds carry different symmetries")
        if not self.has_qnums:
            return Bond(self.dim * other.dim, self.btype)
        degs = {}
        for qa, da in self.sectors:
            for qb, db in other.sectors:
                q = combine_qnums(qa, qb, self.syms)
                degs[q] = degs.get(q, 0) + da * db  # dict keeps first-insertion order
        return Bond(btype=self.btype, sectors=list(degs.items()), syms=self.syms)

    def combine_(self, other):
        from .dense import bump_epoch
        bump_epoch()
        m = self.combine(other)
        self.btype, self.dim, self.sectors, self.syms, self._offsets = m.btype, m.dim, m.sectors, m.syms, None
        return self

    def redirect(self):
        """IN <-> OUT copy; REGULAR bonds are returned unchanged."""
        if self.btype == REGULAR:
            return self
        b = Bond.__new__(Bond)
        b.btype = OUT if self.btype == IN else IN
        b.dim, b.sectors, b.syms, b._offsets = self.dim, self.sectors, self.syms, None
        return b

    def redirect_(self):
        from .dense import bump_epoch
        bump_epoch()
        if self.btype != REGULAR:
            self.btype = OUT if self.btype == IN else IN
        return self

    def __eq__(self, other):
        if not isinstance(other, Bond):
            return NotImplemented
        return (self.btype, self.dim, self.sectors, self.syms) == (other.btype, other.dim, other.sectors, other.syms)

    def __hash__(self):
        return hash((self.btype, self.dim, self.sectors, self.syms))

    def __repr__(self):
        return f"<Bond {self!s}>".replace("\n", " | ")

    def __str__(self):
        tag = {IN: "|IN (KET)>", OUT: "< OUT (BRA)|"}.get(self.btype, "REGULAR")
        lines = [f"Dim = {self.dim} |type: {tag}"]
        if self.has_qnums:
            for i, s in enumerate(self.syms):
                lines.append(f" {s}:: " + " ".join(f"{q[i]:+d}".rjust(4) for q in self.qnums()))
            lines.append("Deg>> " + " ".join(str(d).rjust(4) for d in self.degeneracies()))
        return "\n".join(lines)

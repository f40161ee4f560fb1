"""toomgen -- build-time generator of the straight-line streaming programs the
CUDA kernels run for evaluation (step a2) and interpolation (step a4).

This is PRODUCT build tooling (it emits csrc/generated/*.cuh); it shares
nothing with oracle/.  It uses exact Python integers only to (1) derive each
program from the paper's method and (2) prove, symbolically, that every
division in the program is exact for every integer input and that the
program returns exactly w_0..w_2n.

Method (§3, §4, §6; SURVEY.md §8(c) readings 4, 5, 6, 12):
  * evaluation at homogeneous points (p:q):  U(p,q) = sum_k u_k p^k q^(n-k);
    for a +-pair the even and odd sums E, O are formed once and
    U(+-p/q) = E +- O (Eq. 4.1, 4.3-4.4, SPEC eval_pair);
  * interpolation:
      1. even-odd split of each +-pair (Eqs. 4.5-4.6):
         E = (y+ + y-)/2 = W_e part,  O = (y+ - y-)/2 = odd part;
      2. even half: W_e(z) of degree n through nodes (0:1) [y_0],
         (p^2:q^2) [E] and (1:0) [y_inf]; odd half: W_o(z) of degree n-1
         through nodes (p^2:q^2) [O/(pq)] and the unpaired points, whose
         even part is subtracted once the even coefficients are known;
         for the paper's own point set the odd half is aligned as
         x^2 W_o(x^2) with the extra point (0, 0);
      3. each half: peel the node at infinity (leading coefficient),
         substitute x = t/L (L = lcm of the node denominators) so that all
         nodes are integers, run listing 1 (divided differences,
         PAPER.md:114-120) and listing 2 (Newton -> monomial,
         PAPER.md:154-158) unchanged, divide coefficient k by L^(m-k).
  * every division by d = 2^s * o (o odd) is emitted as an exact 2-adic
    division by o (multiply by o^-1 mod 2^32 with a borrow chain, ref [4])
    followed by an exact right shift by s bits.

Streaming model of the emitted code: every variable is an exact integer held
as an infinite little-endian two's-complement stream of 32-bit limbs.  One
loop step produces one limb of every variable, LSB first.  Linear
combinations and 2-adic divisions are causal; a right shift by s = 32a + r
bits needs a+1 limbs of look-ahead, so its output lags its input by a + (r>0)
steps ("delay").  Operands of different delay are aligned with small register
histories.  Because all values are exact integers, no width bookkeeping is
needed: the first L limbs of an output are its two's-complement
representation for any L.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from math import gcd
from functools import reduce
import random

# ----------------------------------------------------------------- point sets


def _lcm(a, b):
    return a * b // gcd(a, b)


@dataclass
class PointSet:
    name: str
    B: int
    points: list          # list of (p, q), q >= 0, gcd(p, q) = 1; (1, 0) is infinity
    mode: str = "h4"      # "h4" or "paper" (aligned odd half)

    @property
    def n(self):
        return self.B - 1

    @property
    def npoints(self):
        return len(self.points)


def pointset_T3():
    # {0, 1, -1, 2, inf}  (BASELINE.json configs[0])
    return PointSet("T3", 3, [(0, 1), (1, 1), (-1, 1), (2, 1), (1, 0)])


def pointset_T4():
    # {0, +-1, +-2, 1/2 (homogeneous (1:2)), inf}  (BASELINE.json configs[1])
    return PointSet("T4", 4, [(0, 1), (1, 1), (-1, 1), (2, 1), (-2, 1), (1, 2), (1, 0)])


def pointset_paper(B):
    # the paper's own points 0, +-1, +-2, ..., +-2^(n-1)  (§4)
    pts = [(0, 1)]
    for j in range(B - 1):
        pts += [(1 << j, 1), (-(1 << j), 1)]
    return PointSet(f"P{B}", B, pts, mode="paper")


def pointset_T16_31():
    """The 31-point set of configs[4] (SURVEY §8(c) reading 5): 0, inf and
    the 29 smallest-height +-p/q (height max(|p|,q)); within a height by
    min(|p|,q) ascending, |p| > q first, + before -; last point +2/5."""
    cand = []
    for h in range(1, 6):
        fr = []
        for p in range(0, h + 1):
            for q in range(1, h + 1):
                if max(p, q) != h or gcd(p, q) != 1 or p == 0:
                    continue
                fr.append((p, q))
        fr.sort(key=lambda pq: (min(pq), 0 if pq[0] > pq[1] else 1))
        for p, q in fr:
            cand += [(p, q), (-p, q)]
    pts = [(0, 1), (1, 0)] + cand[:29]
    return PointSet("T16", 16, pts)


# ------------------------------------------------------------ program model


@dataclass
class Term:
    var: str
    m: int          # small signed multiplier
    s: int = 0      # left shift in bits (term = m * (var << s))


@dataclass
class Op:
    dst: str
    terms: list
    odiv: int = 1   # exact division by this odd number
    shr: int = 0    # then exact right shift by this many bits
    note: str = ""


@dataclass
class Program:
    name: str
    inputs: list                         # input stream names, in accessor order
    ops: list = field(default_factory=list)
    outputs: list = field(default_factory=list)   # variable names, in output order
    nunk: int = 0                        # number of unknowns the forms are over
    forms: dict = field(default_factory=dict)     # var -> list[int] (linear form)

    def add(self, dst, terms, d=1, note=""):
        """dst = (sum m*var*2^s) / d, d > 0 integer; checks exactness of the
        linear form symbolically and records the op."""
        assert d > 0
        s = (d & -d).bit_length() - 1
        o = d >> s
        form = [0] * self.nunk
        for t in terms:
            f = self.forms[t.var]
            for j in range(self.nunk):
                form[j] += t.m * (f[j] << t.s)
        for j in range(self.nunk):
            if form[j] % d:
                raise AssertionError(f"{self.name}: inexact division by {d} in {dst} ({note})")
            form[j] //= d
        self.forms[dst] = form
        self.ops.append(Op(dst, [Term(t.var, t.m, t.s) for t in terms if t.m != 0], o, s, note))
        return dst


def _norm_terms(terms):
    """Merge identical (var, s) terms; drop zero multipliers; turn large
    power-of-two multipliers into shifts (streams stay 32-bit per term)."""
    acc = {}
    for t in terms:
        m, s = t.m, t.s
        while m != 0 and m % 2 == 0 and abs(m) >= (1 << 20):
            m //= 2
            s += 1
        acc[(t.var, s)] = acc.get((t.var, s), 0) + m
    out = [Term(v, m, s) for (v, s), m in acc.items() if m != 0]
    return out


class _Gen:
    def __init__(self, prog):
        self.p = prog
        self.k = 0

    def new(self, base):
        self.k += 1
        return f"{base}_{self.k}"

    def op(self, base, terms, d=1, note=""):
        terms = _norm_terms(terms)
        # a plain copy needs no op
        if d == 1 and len(terms) == 1 and terms[0].m == 1 and terms[0].s == 0:
            return terms[0].var
        # factor d so that each emitted odd divisor fits one 32-bit word
        s = (d & -d).bit_length() - 1
        o = d >> s
        if o < (1 << 32):
            return self.p.add(self.new(base), terms, d, note)
        # split o into word-sized factors (exact at every stage: all factors
        # divide every coefficient of the form, checked by Program.add)
        facs = _word_factors(o)
        cur = self.p.add(self.new(base), terms, facs[0] << s, note)
        for f in facs[1:]:
            cur = self.p.add(self.new(base), [Term(cur, 1)], f, note + " (cont.)")
        return cur


def _word_factors(o):
    fs = []
    x = o
    p = 3
    primes = []
    while p * p <= x:
        while x % p == 0:
            primes.append(p)
            x //= p
        p += 2
    if x > 1:
        primes.append(x)
    cur = 1
    for q in primes:
        if cur * q >= (1 << 32):
            fs.append(cur)
            cur = 1
        cur *= q
    fs.append(cur)
    return fs


# ------------------------------------------------------------- evaluation


def build_eval(ps: PointSet) -> Program:
    """Evaluate the B blocks u_0..u_n at every point of ps (homogeneous),
    sharing the even and odd sums of each +-pair (Eq. 4.1)."""
    n = ps.n
    prog = Program(f"eval_{ps.name}", [f"u{k}" for k in range(ps.B)], nunk=ps.B)
    for k in range(ps.B):
        prog.forms[f"u{k}"] = [1 if j == k else 0 for j in range(ps.B)]
    g = _Gen(prog)
    pts = ps.points
    done = {}
    for idx, (p, q) in enumerate(pts):
        if idx in done:
            continue
        c = [p**k * q ** (n - k) for k in range(ps.B)]
        partner = None
        if p > 0:
            for j2, (p2, q2) in enumerate(pts):
                if p2 == -p and q2 == q:
                    partner = j2
        if partner is not None:
            E = g.op("E", [Term(f"u{k}", c[k]) for k in range(0, ps.B, 2)], note=f"E({p}/{q})")
            O = g.op("O", [Term(f"u{k}", c[k]) for k in range(1, ps.B, 2)], note=f"O({p}/{q})")
            done[idx] = g.op("Up", [Term(E, 1), Term(O, 1)], note=f"U(+{p}/{q}) = E + O")
            done[partner] = g.op("Um", [Term(E, 1), Term(O, -1)], note=f"U(-{p}/{q}) = E - O")
        else:
            done[idx] = g.op("U", [Term(f"u{k}", c[k]) for k in range(ps.B)], note=f"U({p}:{q})")
    prog.outputs = [done[i] for i in range(len(pts))]
    for i, (p, q) in enumerate(pts):
        assert prog.forms[prog.outputs[i]] == [p**k * q ** (n - k) for k in range(ps.B)]
    return prog


# ---------------------------------------------------------- interpolation


def _solve_half(g: _Gen, nodes, m, tag):
    """nodes: list of (a, b, var) with homogeneous node (a:b) and var holding
    P_h(a, b) = sum_k c_k a^k b^(m-k).  Returns vars c_0..c_m.  (H4 reading
    + the paper's listings.)"""
    assert len(nodes) == m + 1, (tag, len(nodes), m)
    inf = [nd for nd in nodes if nd[1] == 0]
    fin = [nd for nd in nodes if nd[1] != 0]
    cm = None
    if inf:
        assert len(inf) == 1
        cm = inf[0][2]                       # leading coefficient c_m
        peeled = []
        for a, b, v in fin:                  # (v - c_m a^m) / b = P'_h(a, b), degree m-1
            nv = g.op(f"{tag}pk", [Term(v, 1), Term(cm, -(a**m))], b, note=f"peel inf at ({a}:{b})")
            peeled.append((a, b, nv))
        fin = peeled
        m = m - 1
    if m < 0:
        return [cm]
    L = reduce(_lcm, [b for _, b, _ in fin], 1)
    pts = []
    for a, b, v in fin:
        t = a * (L // b)
        f = (L // b) ** m
        if f != 1:
            v = g.op(f"{tag}sc", [Term(v, f)], note=f"scale (L/b)^m at t={t}")
        pts.append((t, v))
    pts.sort(key=lambda tv: tv[0])
    x = [t for t, _ in pts]
    coeff = [v for _, v in pts]
    # listing 1: divided differences, in place, m descending
    for k in range(1, m + 1):
        for mm in range(m, k - 1, -1):
            den = x[mm] - x[mm - k]
            assert den > 0
            coeff[mm] = g.op(f"{tag}a", [Term(coeff[mm], 1), Term(coeff[mm - 1], -1)], den,
                             note=f"listing1 k={k} m={mm}: /(x[{mm}]-x[{mm - k}])")
    # listing 2: Newton -> monomial
    for mm in range(m - 1, -1, -1):
        for k in range(mm, m):
            if x[mm] != 0:
                coeff[k] = g.op(f"{tag}b", [Term(coeff[k], 1), Term(coeff[k + 1], -x[mm])],
                                note=f"listing2 m={mm} k={k}: -= x[{mm}]*coeff[{k + 1}]")
    # undo the substitution x = t/L
    res = []
    for k in range(m + 1):
        dk = L ** (m - k)
        res.append(coeff[k] if dk == 1 else g.op(f"{tag}c", [Term(coeff[k], 1)], dk, note=f"/L^{m - k}"))
    if cm is not None:
        res.append(cm)
    return res


def build_interp(ps: PointSet) -> Program:
    n = ps.n
    d = 2 * n
    pts = ps.points
    prog = Program(f"interp_{ps.name}", [f"y{k}" for k in range(len(pts))], nunk=d + 1)
    for k, (p, q) in enumerate(pts):
        prog.forms[f"y{k}"] = [p**j * q ** (d - j) for j in range(d + 1)]
    g = _Gen(prog)
    zero = [k for k, pq in enumerate(pts) if pq == (0, 1)]
    inf = [k for k, pq in enumerate(pts) if pq == (1, 0)]
    pairs, unpaired = [], []
    used = set(zero + inf)
    for k, (p, q) in enumerate(pts):
        if k in used or p <= 0:
            continue
        m = [j for j, pq in enumerate(pts) if pq == (-p, q)]
        if m:
            pairs.append((k, m[0], p, q))
            used |= {k, m[0]}
    unpaired = [k for k in range(len(pts)) if k not in used]

    # 1. even-odd split (Eqs. 4.5-4.6)
    EO = []
    for kp, km, p, q in pairs:
        E = g.op("E", [Term(f"y{kp}", 1), Term(f"y{km}", 1)], 2, note=f"W_e: (W({p}/{q})+W(-{p}/{q}))/2 (Eq. 4.5)")
        EO.append((p, q, E, kp, km))

    # 2. even half: c_k = w_{2k}, degree n
    nodes = []
    if zero:
        nodes.append((0, 1, f"y{zero[0]}"))
    for p, q, E, _, _ in EO:
        nodes.append((p * p, q * q, E))
    if inf:
        nodes.append((1, 0, f"y{inf[0]}"))
    even = _solve_half(g, nodes, n, "e")

    # 3. odd half: c'_k = w_{2k+1}, degree n-1
    if ps.mode == "paper":
        assert not unpaired and not inf
        # x^2 W_o(x^2) = x (W(x) - W(-x)) / 2, plus the point (0, 0)
        nodes = []
        for p, q, E, kp, km in EO:
            assert q == 1
            v = g.op("Ox", [Term(f"y{kp}", p), Term(f"y{km}", -p)], 2, note=f"x^2 W_o(x^2) at x={p} (Eq. 4.6 * x^2)")
            nodes.append((p * p, 1, v))
        # the extra point (0, 0): a zero stream
        prog.forms["ZERO"] = [0] * (d + 1)
        nodes.insert(0, (0, 1, "ZERO"))
        odd_aligned = _solve_half(g, nodes, n, "o")
        odd = odd_aligned[1:]      # "the resulting coefficients move one place higher"
    else:
        nodes = []
        for p, q, E, kp, km in EO:
            v = g.op("O", [Term(f"y{kp}", 1), Term(f"y{km}", -1)], 2 * p * q, note=f"W_o node: (W(+)-W(-))/(2pq) at {p}/{q}")
            nodes.append((p * p, q * q, v))
        for k in unpaired:
            p, q = pts[k]
            # y - even part, divided by p q: the odd polynomial's homogeneous value
            terms = [Term(f"y{k}", 1)]
            for kk in range(n + 1):
                terms.append(Term(even[kk], -(p ** (2 * kk)) * q ** (d - 2 * kk)))
            v = g.op("U", terms, p * q, note=f"unpaired {p}/{q}: (y - even part)/(pq)")
            assert p > 0, "unpaired points must be positive"
            nodes.append((p * p, q * q, v))
        odd = _solve_half(g, nodes, n - 1, "o")

    outs = []
    for j in range(d + 1):
        outs.append(even[j // 2] if j % 2 == 0 else odd[j // 2])
    prog.outputs = outs
    for j in range(d + 1):
        f = prog.forms[outs[j]]
        assert f == [1 if i == j else 0 for i in range(d + 1)], (ps.name, j, f)
    return prog


# --------------------------------------------------------- exact simulation


def run_program(prog: Program, inputs: dict) -> list:
    """Execute the program on exact Python ints (whole values, not streams)."""
    env = dict(inputs)
    env["ZERO"] = 0
    for op in prog.ops:
        s = 0
        for t in op.terms:
            s += t.m * (env[t.var] << t.s)
        d = op.odiv << op.shr
        assert s % d == 0, f"inexact {op.dst}"
        env[op.dst] = s // d
    return [env[v] for v in prog.outputs]


def selfcheck(ps: PointSet, trials=20, bits=300, seed=1):
    """Round trip on random signed block polynomials: eval -> products ->
    interp must return the block convolution w_k = sum u_i v_j."""
    rng = random.Random(seed)
    ev, it = build_eval(ps), build_interp(ps)
    for _ in range(trials):
        U = [rng.randrange(-(1 << bits), 1 << bits) for _ in range(ps.B)]
        V = [rng.randrange(-(1 << bits), 1 << bits) for _ in range(ps.B)]
        EU = run_program(ev, {f"u{k}": U[k] for k in range(ps.B)})
        EV = run_program(ev, {f"u{k}": V[k] for k in range(ps.B)})
        Y = {f"y{k}": EU[k] * EV[k] for k in range(ps.npoints)}
        W = run_program(it, Y)
        conv = [sum(U[i] * V[k - i] for i in range(ps.B) if 0 <= k - i < ps.B) for k in range(2 * ps.B - 1)]
        assert W == conv, ps.name
    return True


# ------------------------------------------------------------------ emitter


def _inv32(o):
    return pow(o, -1, 1 << 32)


def _live_ops(prog, outputs):
    need = set(outputs)
    ops = []
    for op in reversed(prog.ops):
        if op.dst in need:
            ops.append(op)
            for t in op.terms:
                need.add(t.var)
    ops.reverse()
    return ops


def fuse_single_use(prog: Program, max_mult=1 << 24) -> Program:
    """Inline every op whose result is used exactly once (and is not an
    output) into its consumer:  Y = (c*X*2^t + R)/dY with X = N_X/dX  becomes
    Y = (c*2^t*N_X + dX*R)/(dX*dY).  The merged op is re-checked for exactness
    by Program.add's symbolic form test; merges that would need a divisor odd
    part >= 2^32 or multipliers above `max_mult` are skipped."""
    ops = list(prog.ops)
    changed = True
    while changed:
        changed = False
        uses = {}
        for op in ops:
            for t in op.terms:
                uses[t.var] = uses.get(t.var, 0) + 1
        outs = set(prog.outputs)
        byname = {op.dst: op for op in ops}
        for y in ops:
            for t in y.terms:
                x = byname.get(t.var)
                if x is None or t.var in outs or uses.get(t.var, 0) != 1:
                    continue
                dX = x.odiv << x.shr
                terms = []
                for u in y.terms:
                    if u is t:
                        for a in x.terms:
                            terms.append(Term(a.var, t.m * a.m, t.s + a.s))
                    else:
                        terms.append(Term(u.var, u.m * dX, u.s))
                terms = _norm_terms(terms)
                o = x.odiv * y.odiv
                if o >= (1 << 32) or any(abs(u.m) > max_mult for u in terms):
                    continue
                if sum(abs(u.m) for u in terms) >= (1 << 30):
                    continue
                # exactness re-check through the symbolic forms
                form = [0] * prog.nunk
                for u in terms:
                    f = prog.forms[u.var]
                    for j in range(prog.nunk):
                        form[j] += u.m * (f[j] << u.s)
                d = (o << (x.shr + y.shr))
                if any(v % d for v in form) or [v // d for v in form] != prog.forms[y.dst]:
                    continue
                new = Op(y.dst, terms, o, x.shr + y.shr, y.note + " <- " + x.note)
                ops = [new if op is y else op for op in ops if op is not x]
                changed = True
                break
            if changed:
                break
    out = Program(prog.name, prog.inputs, ops, prog.outputs, prog.nunk, prog.forms)
    return out


def input_forms(prog: Program) -> dict:
    """Symbolic execution over the INPUT streams: var -> {input: Fraction}."""
    env = {v: {v: Fraction(1)} for v in prog.inputs}
    env["ZERO"] = {}
    for op in prog.ops:
        acc = {}
        for t in op.terms:
            for k, c in env[t.var].items():
                acc[k] = acc.get(k, 0) + c * t.m * (1 << t.s)
        d = op.odiv << op.shr
        env[op.dst] = {k: Fraction(c) / d for k, c in acc.items() if c != 0}
    return env


def per_output_programs(prog: Program, name: str) -> list:
    """PAPER.md:162 ("for specific n the computation of the c_l can be
    optimized from the entries of this inverse matrix"): compose the whole
    listing program into ONE op per output, w_j = (sum_k A_jk y_k) / D_j,
    with the composition done symbolically from the even-odd + Newton
    program (so A/D are exactly the paper-method's inverse rows).  Each output
    can then be streamed independently (one thread per coefficient)."""
    env = input_forms(prog)
    progs = []
    for j, v in enumerate(prog.outputs):
        form = env[v]
        D = 1
        for c in form.values():
            D = _lcm(D, c.denominator)
        p = Program(f"{name}_w{j}", prog.inputs, nunk=prog.nunk)
        p.forms = dict(prog.forms)
        terms = [Term(k, int(c * D)) for k, c in sorted(form.items(), key=lambda kc: prog.inputs.index(kc[0]))]
        if D == 1 and len(terms) == 1 and terms[0].m == 1:
            p.outputs = [terms[0].var]
        else:
            s = (D & -D).bit_length() - 1
            assert (D >> s) < (1 << 32) and sum(abs(t.m) for t in terms) < (1 << 30), (name, j)
            p.add(f"w{j}", terms, D, note=f"w_{j} = (sum A_jk y_k)/{D}")
            p.outputs = [f"w{j}"]
        assert p.forms[p.outputs[0]] == prog.forms[v]
        progs.append(p)
    return progs


def build_eval_direct(ps: PointSet) -> list:
    """One single-op program per point: U(p:q) = sum_k p^k q^(n-k) u_k."""
    n = ps.n
    progs = []
    for idx, (p, q) in enumerate(ps.points):
        prog = Program(f"eval_{ps.name}_p{idx}", [f"u{k}" for k in range(ps.B)], nunk=ps.B)
        for k in range(ps.B):
            prog.forms[f"u{k}"] = [1 if j == k else 0 for j in range(ps.B)]
        terms = _norm_terms([Term(f"u{k}", p**k * q ** (n - k)) for k in range(ps.B)])
        if len(terms) == 1 and terms[0].m == 1 and terms[0].s == 0:
            prog.outputs = [terms[0].var]
        else:
            prog.add(f"U{idx}", terms, 1, note=f"U({p}:{q})")
            prog.outputs = [f"U{idx}"]
        progs.append(prog)
    return progs


def emit_stream_function(prog: Program, fname: str, outputs=None, out_index=None, prefetch=2, unrolled=False) -> str:
    """Emit a __host__ __device__ template that streams the program LSB-first.

    template <class In, class Out>
    TG_HD void fname(const In& in, Out& out, int nsteps)

    in.load(k, i)   -> uint32 limb i of input k (sign/zero extension done by In)
                       (called for i up to nsteps + maxdelay + prefetch)
    out.store(j, i, x) stores limb i of output j; called for i in [0, nsteps),
                    with i ascending.
    Inputs are software-prefetched `prefetch` steps ahead in registers so the
    global-memory latency overlaps the arithmetic of the current step.
    Per op:  lin (int64, two's complement in a uint64) = carry + sum m_j x_j,
    one IMAD.WIDE.U32 per positive term (tg_madw), IMAD.WIDE + IADD per
    negative term; t = lo(lin), carry = lin >> 32 (arithmetic); then the 2-adic
    exact division by the odd part and the funnel-shift right.
    """
    outputs = list(prog.outputs if outputs is None else outputs)
    out_index = list(range(len(outputs))) if out_index is None else out_index
    ops = _live_ops(prog, outputs)
    for op in ops:
        assert sum(abs(t.m) for t in op.terms) < (1 << 30), (prog.name, op.dst, op.terms)
    delay = {v: 0 for v in prog.inputs}
    delay["ZERO"] = 0
    opD = {}
    for op in ops:
        D = max(delay[t.var] for t in op.terms) if op.terms else 0
        opD[op.dst] = D
        a, r = op.shr // 32, op.shr % 32
        delay[op.dst] = D + a + (1 if r else 0)
    hist = {v: 0 for v in delay}

    def lagof(var, D, s):
        a, r = s // 32, s % 32
        return D - delay[var] + a + (1 if r else 0)

    for op in ops:
        D = opD[op.dst]
        for t in op.terms:
            hist[t.var] = max(hist[t.var], lagof(t.var, D, t.s))
    used_inputs = sorted({t.var for op in ops for t in op.terms if t.var in prog.inputs} |
                         {v for v in outputs if v in prog.inputs}, key=lambda v: prog.inputs.index(v))
    maxdelay = max([delay[v] for v in outputs] + [0])

    def cname(v):
        return v.replace("-", "m")

    L = []
    L.append(f"// generated by toomgen.py from {prog.name}; {len(ops)} ops, max delay {maxdelay}")
    L.append(f"constexpr int {fname}_maxdelay = {maxdelay};")
    if unrolled:
        # compile-time step count, fully unrolled: outputs may land in registers
        prefetch = 0
        L.append("template <int NSTEPS, class In, class Out>")
        L.append(f"TG_HD TG_INLINE void {fname}(const In& in, Out& out) {{")
        L.append("  constexpr int nsteps = NSTEPS;")
    else:
        L.append("template <class In, class Out>")
        L.append(f"TG_HD TG_INLINE void {fname}(const In& in, Out& out, int nsteps) {{")
    vars_all = used_inputs + [op.dst for op in ops]
    for v in vars_all:
        for h in range(1, hist[v] + 1):
            L.append(f"  uint32_t {cname(v)}_h{h} = 0u;")
    for op in ops:
        L.append(f"  uint64_t {cname(op.dst)}_acc = 0ull;")
        if op.odiv != 1:
            L.append(f"  uint32_t {cname(op.dst)}_bor = 0u;")
        if op.shr % 32:
            L.append(f"  uint32_t {cname(op.dst)}_qp = 0u;")
    # prefetch registers
    for v in used_inputs:
        k = prog.inputs.index(v)
        for p in range(prefetch):
            L.append(f"  uint32_t {cname(v)}_pf{p} = in.load({k}, {p});")
    if unrolled:
        L.append(f"  constexpr int total = nsteps + {maxdelay};")
        L.append("  #pragma unroll")
    else:
        L.append(f"  const int total = nsteps + {maxdelay};")
        L.append("  #pragma unroll 1")
    L.append("  for (int i = 0; i < total; ++i) {")
    for v in used_inputs:
        k = prog.inputs.index(v)
        if prefetch == 0:
            L.append(f"    const uint32_t {cname(v)}_h0 = in.load({k}, i);")
            continue
        L.append(f"    const uint32_t {cname(v)}_h0 = {cname(v)}_pf0;")
        for p in range(prefetch - 1):
            L.append(f"    {cname(v)}_pf{p} = {cname(v)}_pf{p + 1};")
        L.append(f"    {cname(v)}_pf{prefetch - 1} = in.load({k}, i + {prefetch});")
    for op in ops:
        D = opD[op.dst]
        dn = cname(op.dst)
        L.append(f"    // {op.dst} = ({' + '.join(f'{t.m}*{t.var}<<{t.s}' for t in op.terms)}) / {op.odiv << op.shr}   [{op.note}]")
        L.append(f"    uint32_t {dn}_h0;")
        L.append("    {")
        srcs = []
        for t in op.terms:
            if t.var == "ZERO":
                continue
            lag = lagof(t.var, D, t.s)
            r = t.s % 32
            vn = cname(t.var)
            if r == 0:
                src = f"{vn}_h{lag}"
            else:
                src = f"tg_shl_limb({vn}_h{lag}, {vn}_h{lag - 1}, {r})"
            srcs.append((src, t.m))
        # independent mad.wide chains, the carry of the previous limb last
        L += _lincomb_lines(srcs, f"{dn}_acc", "lin", "      ")
        L.append(f"      uint32_t t = (uint32_t)lin;")
        L.append(f"      {dn}_acc = (uint64_t)((int64_t)lin >> 32);")
        if op.odiv != 1:
            L.append(f"      t = tg_divexact_step(t, {dn}_bor, 0x{_inv32(op.odiv):08X}u, {op.odiv}u);   // / {op.odiv}")
        r = op.shr % 32
        if r:
            L.append(f"      {dn}_h0 = tg_shr_limb({dn}_qp, t, {r});")
            L.append(f"      {dn}_qp = t;")
        else:
            L.append(f"      {dn}_h0 = t;")
        L.append("    }")
    for j, v in zip(out_index, outputs):
        dv = delay[v]
        vn = cname(v)
        if v == "ZERO":
            L.append(f"    if (i < nsteps) out.store({j}, i, 0u);")
        elif dv == 0:
            L.append(f"    if (i < nsteps) out.store({j}, i, {vn}_h0);")
        else:
            L.append(f"    if (i >= {dv} && i - {dv} < nsteps) out.store({j}, i - {dv}, {vn}_h0);")
    for v in vars_all:
        for h in range(hist[v], 0, -1):
            L.append(f"    {cname(v)}_h{h} = {cname(v)}_h{h - 1};")
    L.append("  }")
    L.append("}")
    return "\n".join(L)


def emit_row_tables(ps: PointSet) -> str:
    """Constant tables for the fused kernel's table-driven streams:
    evaluation coefficients c[k][j] = p_k^j q_k^(n-j) (homogeneous points) and
    the interpolation rows w_j = (sum_k A[j][k] y_k) / (o_j 2^s_j), composed
    from the even-odd + Newton-listing program (per_output_programs)."""
    n = ps.n
    NP = ps.npoints
    rows = per_output_programs(build_interp(ps), f"interp_{ps.name}")
    L = [f"// ---- table-driven rows for {ps.name} (fused bottom-level kernel)"]
    L.append(f"TG_CONST long long tg_evalc_{ps.name}[{NP}][{ps.B}] = {{")
    for (p, q) in ps.points:
        L.append("  {" + ", ".join(str(p**j * q ** (n - j)) for j in range(ps.B)) + "},")
    L.append("};")
    # the same coefficients as a constexpr function (compile-time point index)
    L.append(f"TG_HD constexpr long long tg_evalc_cx_{ps.name}(int k, int j) {{")
    L.append(f"  return")
    for k, (p, q) in enumerate(ps.points):
        for j in range(ps.B):
            L.append(f"    (k == {k} && j == {j}) ? {p**j * q ** (n - j)}ll :")
    L.append("    0ll;")
    L.append("}")
    A, O, INV, S = [], [], [], []
    for j, pr in enumerate(rows):
        coef = [0] * NP
        if pr.ops:
            op = pr.ops[0]
            for t in op.terms:
                assert t.s == 0
                coef[pr.inputs.index(t.var)] = t.m
            o, s = op.odiv, op.shr
        else:
            coef[pr.inputs.index(pr.outputs[0])] = 1
            o, s = 1, 0
        assert s < 32
        A.append(coef)
        O.append(o)
        INV.append(_inv32(o))
        S.append(s)
    L.append(f"TG_CONST long long tg_rowA_{ps.name}[{NP}][{NP}] = {{")
    for r in A:
        L.append("  {" + ", ".join(str(x) for x in r) + "},")
    L.append("};")
    L.append(f"TG_CONST unsigned tg_rowO_{ps.name}[{NP}] = {{" + ", ".join(f"{x}u" for x in O) + "};")
    L.append(f"TG_CONST unsigned tg_rowInv_{ps.name}[{NP}] = {{" + ", ".join(f"0x{x:08X}u" for x in INV) + "};")
    L.append(f"TG_CONST int tg_rowS_{ps.name}[{NP}] = {{" + ", ".join(str(x) for x in S) + "};")
    # scan constants of the instance-resident level kernels (csrc/level34.cuh,
    # RES_CH = 9 positions per thread): 2^32 mod o, Mch = 2^(32*9) mod o and
    # its inverse (all o here are odd, > 1 or the no-division marker 1)
    RES_CH = 9
    P32 = [(1 << 32) % o if o > 1 else 0 for o in O]
    MCH = [pow(2, 32 * RES_CH, o) if o > 1 else 0 for o in O]
    MI = [pow(m, -1, o) if o > 1 else 0 for m, o in zip(MCH, O)]
    L.append(f"TG_CONST unsigned tg_rowP32_{ps.name}[{NP}] = {{" + ", ".join(f"{x}u" for x in P32) + "};")
    L.append(f"TG_CONST unsigned tg_rowMch9_{ps.name}[{NP}] = {{" + ", ".join(f"{x}u" for x in MCH) + "};")
    L.append(f"TG_CONST unsigned tg_rowMi9_{ps.name}[{NP}] = {{" + ", ".join(f"{x}u" for x in MI) + "};")
    # combined form over a common denominator Dc = lcm_j D_j (PAPER.md:162
    # matrix form + Eq. 1.3): Dc w = sum_j 2^(32 b j) sum_k (Dc/D_j) A[j][k] y_k
    Ds = [O[j] << S[j] for j in range(NP)]
    Dc = reduce(_lcm, Ds, 1)
    sc = (Dc & -Dc).bit_length() - 1
    oc = Dc >> sc
    assert oc < (1 << 32) and sc < 32
    L.append(f"TG_CONST long long tg_combA_{ps.name}[{NP}][{NP}] = {{")
    for j in range(NP):
        L.append("  {" + ", ".join(str(A[j][k] * (Dc // Ds[j])) for k in range(NP)) + "},")
    L.append("};")
    L.append(f"constexpr unsigned tg_combO_{ps.name} = {oc}u;")
    L.append(f"constexpr unsigned tg_combInv_{ps.name} = 0x{_inv32(oc):08X}u;")
    L.append(f"constexpr int tg_combS_{ps.name} = {sc};")
    # the combined rows as a constexpr function (lazy long levels, csrc/lazy.cuh)
    L.append(f"TG_HD constexpr long long tg_combA_cx_{ps.name}(int j, int k) {{")
    L.append(f"  return")
    for j in range(NP):
        for k in range(NP):
            c = A[j][k] * (Dc // Ds[j])
            if c:
                L.append(f"    (j == {j} && k == {k}) ? {c}ll :")
    L.append("    0ll;")
    L.append("}")
    return "\n".join(L)


def _lincomb_lines(terms, acc, out, ind="  "):
    """C lines computing out = acc + sum_k m_k * y_k (mod 2^64) with the
    products spread over up to four independent mad.wide chains (two for
    positive, two for negative multipliers) instead of one serial chain, so
    the multiply-adds of one limb overlap."""
    pos = [(y, m) for y, m in terms if m > 0]
    neg = [(y, -m) for y, m in terms if m < 0]
    L = []
    chains = []
    for tag, grp in (("p", pos), ("n", neg)):
        for c in range(2):
            sub = grp[c::2]
            if not sub:
                continue
            name = f"_{tag}{c}"
            L.append(f"{ind}uint64_t {name} = 0ull;")
            for y, m in sub:
                L.append(f"{ind}{name} = tg_madw({m}u, {y}, {name});")
            chains.append((tag, name))
    # the carry from the previous limb enters last: it is the only input on the
    # limb-to-limb critical path
    expr = " + ".join([n for t, n in chains if t == "p"] + [acc])
    negs = [n for t, n in chains if t == "n"]
    if negs:
        expr = f"({expr}) - ({' + '.join(negs)})"
    L.append(f"{ind}const uint64_t {out} = {expr};")
    return L


def emit_row_functions(ps: PointSet) -> str:
    """Specialised per-coefficient streams for the fused kernel's phase B:
    w_j = (sum_k A_jk y_k) / (o_j 2^s_j) with immediate multipliers and only
    the nonzero terms; y_k in smem at Y[(k*w2 + t)*32], w_j to dst[t*32].
    Requires w2 > Lw (child products are wider than the coefficients), so no
    sign fill is ever needed.  Rows that are plain copies (w_0 = y_0,
    w_2n = y_inf) are not emitted."""
    rows = per_output_programs(build_interp(ps), f"interp_{ps.name}")
    L = [f"// ---- specialised coefficient rows for {ps.name}"]
    # Toom-4 rows rolled (the C2 fused kernel is instruction-cache bound:
    # 519 -> 486 us); Toom-3 rows unrolled by 2 (C1: 27 vs 32 us)
    u = 1 if ps.B >= 4 else 2
    L.append(f"#ifndef TG_ROW_UNROLL_{ps.name}")
    L.append(f'#  define TG_ROW_UNROLL_{ps.name} _Pragma("unroll {u}")')
    L.append("#endif")
    for j, pr in enumerate(rows):
        if not pr.ops:
            continue
        op = pr.ops[0]
        idx = [(pr.inputs.index(t.var), t.m) for t in op.terms]
        assert all(t.s == 0 for t in op.terms) and op.shr < 32
        L.append(f"// w_{j} = ({' '.join(f'{m:+d}*y{k}' for k, m in idx)}) / {op.odiv << op.shr}")
        # W2 (the child product width) is a template parameter so that the
        # row offsets k*W2*32 fold into the shared-memory load immediates
        L.append(f"template <int W2> __device__ __forceinline__ void tg_row_{ps.name}_{j}(const uint32_t* __restrict__ Y, uint32_t* __restrict__ dst, int Lw) {{")
        L.append("  uint64_t acc = 0; uint32_t qp = 0;")
        if op.odiv != 1:
            L.append("  uint32_t bor = 0;")
        # one position: loads, linear combination, carry, exact division
        # (Toom-4: position 0 peeled so that the loop stores unconditionally)
        L.append("  auto step = [&](int t) -> uint32_t {")
        L.append("    const uint32_t* __restrict__ yt = Y + t * 32;")
        for k, m in idx:
            L.append(f"    const uint32_t y{k} = yt[{k} * W2 * 32];")
        L += _lincomb_lines([(f"y{k}", m) for k, m in idx], "acc", "lin", "    ")
        L.append("    acc = (uint64_t)((int64_t)lin >> 32);")
        if op.odiv != 1:
            L.append(f"    return tg_divexact_step((uint32_t)lin, bor, 0x{_inv32(op.odiv):08X}u, {op.odiv}u);")
        else:
            L.append("    return (uint32_t)lin;")
        L.append("  };")
        bor = "bor" if op.odiv != 1 else "0u"
        if ps.B >= 4:
            # peeled (C2 fused 426 -> 418 us)
            L.append("  qp = step(0);")
            L.append(f"  TG_CHECK_LOW(qp, {op.shr});")
            L.append(f"  TG_ROW_UNROLL_{ps.name}")
            L.append("  for (int t = 1; t <= Lw; ++t) {")
            L.append("    const uint32_t q = step(t);")
            L.append(f"    dst[(t - 1) * 32] = tg_shr_limb_or_delay(qp, q, {op.shr});")
            L.append("    qp = q;")
            L.append("  }")
        else:
            # (peeling measured slower for the unrolled Toom-3 rows: C1, C3)
            L.append(f"  TG_ROW_UNROLL_{ps.name}")
            L.append("  for (int t = 0; t <= Lw; ++t) {")
            L.append("    const uint32_t q = step(t);")
            L.append(f"    if (t > 0) dst[(t - 1) * 32] = tg_shr_limb_or_delay(qp, q, {op.shr});")
            L.append(f"    else TG_CHECK_LOW(q, {op.shr});")
            L.append("    qp = q;")
            L.append("  }")
        # debug exactness check: after the last position the
        # value D_j w_j is fully sign-extended, so the carry is 0 / -1 and the
        # 2-adic borrow 0 / o-1 exactly when the division was exact
        # (the y_k are read mod 2^(32 W2): a negative y_k adds -A_k 2^(32 W2)
        # to the true dividend, so the carry is corrected by its sign)
        L.append("  if (TG_CHECK_ENABLED) {")
        L.append("    uint64_t corr = 0;")
        for k, m in idx:
            L.append(f"    corr += (uint64_t)({m}ll) * (Y[({k} * W2 + W2 - 1) * 32] >> 31);")
        L.append(f"    TG_CHECK_END(acc - corr, {bor}, {op.odiv}u);")
        L.append("  }")
        L.append("}")
    return "\n".join(L)


def emit_rowstep_functions(ps: PointSet) -> str:
    """One LSB-first step of each nontrivial coefficient row: given limb t of
    every y_k, update the row's carry / borrow state and return limb t-1 of
    w_j (the exact shift lags one limb).  Callers choose where y and w live."""
    rows = per_output_programs(build_interp(ps), f"interp_{ps.name}")
    NP = ps.npoints
    L = [f"// ---- coefficient row steps for {ps.name}"]
    for j, pr in enumerate(rows):
        if not pr.ops:
            continue
        op = pr.ops[0]
        idx = [(pr.inputs.index(t.var), t.m) for t in op.terms]
        L.append(f"__device__ __forceinline__ uint32_t tg_rowstep_{ps.name}_{j}(const uint32_t (&y)[{NP}], tg_rowstate& st) {{")
        L += _lincomb_lines([(f"y[{k}]", m) for k, m in idx], "st.acc", "lin", "  ")
        L.append("  st.acc = (uint64_t)((int64_t)lin >> 32);")
        if op.odiv != 1:
            L.append(f"  const uint32_t q = tg_divexact_step((uint32_t)lin, st.bor, 0x{_inv32(op.odiv):08X}u, {op.odiv}u);")
        else:
            L.append("  const uint32_t q = (uint32_t)lin;")
        L.append(f"  const uint32_t r = tg_shr_limb_or_delay(st.qp, q, {op.shr});")
        L.append("  st.qp = q;")
        L.append("  return r;")
        L.append("}")
    L.append(f"__device__ __forceinline__ uint32_t tg_rowstep_{ps.name}(int j, const uint32_t (&y)[{NP}], tg_rowstate& st) {{")
    L.append("  switch (j) {")
    for j, pr in enumerate(rows):
        if pr.ops:
            L.append(f"    case {j}: return tg_rowstep_{ps.name}_{j}(y, st);")
        else:
            k = pr.inputs.index(pr.outputs[0])
            L.append(f"    case {j}: {{ const uint32_t r = st.qp; st.qp = y[{k}]; return r; }}")
    L.append("  }")
    L.append("  return 0u;")
    L.append("}")
    return "\n".join(L)


def emit_evalrow_functions(ps: PointSet) -> str:
    """Specialised per-point evaluation streams for the fused kernel's phase A:
    U(p:q) = sum_j p^j q^(n-j) u_j for BOTH operands in one rolled loop, with
    immediate multipliers.  Parent blocks are staged in smem padded to E limbs
    (zero / sign filled), block j limb t at P[(j*E + t)*33]; the two E-limb
    results go to dU[t*32], dV[t*32]."""
    n = ps.n
    L = [f"// ---- specialised point evaluations for {ps.name}"]
    u = 1 if ps.B >= 4 else 2   # as the rows (instruction cache of the Toom-4 fused kernel)
    L.append(f"#ifndef TG_EVALROW_UNROLL_{ps.name}")
    L.append(f'#  define TG_EVALROW_UNROLL_{ps.name} _Pragma("unroll {u}")')
    L.append("#endif")
    for k, (p, q) in enumerate(ps.points):
        coef = [p**j * q ** (n - j) for j in range(ps.B)]
        terms = [(j, c) for j, c in enumerate(coef) if c != 0]
        L.append(f"// U({p}:{q}) = {' '.join(f'{c:+d}*u{j}' for j, c in terms)}")
        L.append(f"template <int E> __device__ __forceinline__ void tg_evalrow_{ps.name}_{k}("
                 "const uint32_t* __restrict__ PU, const uint32_t* __restrict__ PV, uint32_t* __restrict__ dU, uint32_t* __restrict__ dV) {")
        if len(terms) == 1 and terms[0][1] == 1:
            j = terms[0][0]
            L.append("  #pragma unroll 2")
            L.append(f"  for (int t = 0; t < E; ++t) {{ dU[t * 32] = PU[({j} * E + t) * 33]; dV[t * 32] = PV[({j} * E + t) * 33]; }}")
            L.append("}")
            continue
        L.append("  uint64_t au = 0, av = 0;")
        L.append(f"  TG_EVALROW_UNROLL_{ps.name}")
        L.append("  for (int t = 0; t < E; ++t) {")
        L.append("    uint64_t lu = au, lv = av;")
        for j, c in terms:
            L.append(f"    {{ const uint32_t x = PU[({j} * E + t) * 33], y = PV[({j} * E + t) * 33];")
            if c > 0:
                L.append(f"      lu = tg_madw({c}u, x, lu); lv = tg_madw({c}u, y, lv); }}")
            else:
                L.append(f"      lu = tg_msubw({-c}u, x, lu); lv = tg_msubw({-c}u, y, lv); }}")
        L.append("    dU[t * 32] = (uint32_t)lu; dV[t * 32] = (uint32_t)lv;")
        L.append("    au = (uint64_t)((int64_t)lu >> 32); av = (uint64_t)((int64_t)lv >> 32);")
        L.append("  }")
        L.append("}")
    # register versions (fully unrolled): the evaluated operands go straight
    # into the product's register arrays
    for k, (p, q) in enumerate(ps.points):
        coef = [p**j * q ** (n - j) for j in range(ps.B)]
        terms = [(j, c) for j, c in enumerate(coef) if c != 0]
        L.append(f"template <int E> __device__ __forceinline__ void tg_evalreg_{ps.name}_{k}("
                 "const uint32_t* __restrict__ PU, const uint32_t* __restrict__ PV, uint32_t (&a)[E], uint32_t (&b)[E]) {")
        L.append("  uint64_t au = 0, av = 0;")
        L.append("  #pragma unroll")
        L.append("  for (int t = 0; t < E; ++t) {")
        L.append("    uint64_t lu = au, lv = av;")
        for j, c in terms:
            L.append(f"    {{ const uint32_t x = PU[({j} * E + t) * 33], y = PV[({j} * E + t) * 33];")
            if c > 0:
                L.append(f"      lu = tg_madw({c}u, x, lu); lv = tg_madw({c}u, y, lv); }}")
            else:
                L.append(f"      lu = tg_msubw({-c}u, x, lu); lv = tg_msubw({-c}u, y, lv); }}")
        L.append("    a[t] = (uint32_t)lu; b[t] = (uint32_t)lv;")
        L.append("    au = (uint64_t)((int64_t)lu >> 32); av = (uint64_t)((int64_t)lv >> 32);")
        L.append("  }")
        L.append("}")
    return "\n".join(L)


def stats(prog: Program):
    nterms = sum(len(op.terms) for op in prog.ops)
    ndiv = sum(1 for op in prog.ops if op.odiv != 1)
    nshr = sum(1 for op in prog.ops if op.shr)
    return dict(ops=len(prog.ops), terms=nterms, odd_divisions=ndiv, shifts=nshr)


HEADER = """// AUTO-GENERATED by paper_1602_02740_b200/gen/toomgen.py -- do not edit.
// Streaming evaluation / interpolation programs (PAPER.md §3, §4, §6;
// see toomgen.py docstring for the method and the streaming model).
#pragma once
#include <stdint.h>
#ifndef TG_HD
#  ifdef __CUDACC__
#    define TG_HD __host__ __device__
#    define TG_INLINE __forceinline__
#  else
#    define TG_HD
#    define TG_INLINE inline
#  endif
#endif
#ifndef TG_CONST
#  ifdef __CUDACC__
#    define TG_CONST __constant__
#  else
#    define TG_CONST static const
#  endif
#endif
// optional exact-division checks (defined by the CUDA library, csrc/check.cuh;
// no-ops elsewhere)
#ifndef TG_CHECK_LOW
#  define TG_CHECK_LOW(q0, s) ((void)0)
#endif
#ifndef TG_CHECK_END
#  define TG_CHECK_END(acc, bor, o) ((void)0)
#endif
#ifndef TG_CHECK_ENABLED
#  define TG_CHECK_ENABLED 0
#endif
#ifndef TG_HELPERS_DEFINED
#define TG_HELPERS_DEFINED
struct tg_rowstate { uint64_t acc; uint32_t bor, qp; };
TG_HD TG_INLINE uint32_t tg_mulhi(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}
// lin + m*x (64-bit accumulate; one IMAD.WIDE.U32 on the device: written in
// C, ptxas fuses the add into the IMAD.WIDE; an inline mad.wide.u32 was split
// into a zero-addend IMAD.WIDE + IADD3 + IMAD.X)
TG_HD TG_INLINE uint64_t tg_madw(uint32_t m, uint32_t x, uint64_t lin) {
  return lin + (uint64_t)m * x;
}
// lin - m*x (mod 2^64): (2^32 - m)*x + lin - x*2^32
TG_HD TG_INLINE uint64_t tg_msubw(uint32_t m, uint32_t x, uint64_t lin) {
#ifdef __CUDA_ARCH__
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(0u - m), "r"(x), "l"(lin));
  return r - ((uint64_t)x << 32);
#else
  return lin - (uint64_t)m * x;
#endif
}
// one limb of the 2-adic exact division by odd o (ref [4]): q = (t - bor) * o^-1,
// bor' = hi(q*o) + (t < bor)
TG_HD TG_INLINE uint32_t tg_divexact_step(uint32_t t, uint32_t& bor, uint32_t oinv, uint32_t o) {
#if defined(__CUDA_ARCH__) && !defined(TG_DIVEXACT_C)
  // sub.cc's borrow-out feeds subc (bb = -borrow); bor' = hi(q o) + borrow
  uint32_t q, nb;
  asm("{\\n\\t.reg .u32 x, bb;\\n\\t"
      "sub.cc.u32 x, %2, %3;\\n\\t"
      "subc.u32 bb, 0, 0;\\n\\t"
      "mul.lo.u32 %0, x, %4;\\n\\t"
      "mul.hi.u32 %1, %0, %5;\\n\\t"
      "sub.u32 %1, %1, bb;\\n\\t}"
      : "=r"(q), "=r"(nb) : "r"(t), "r"(bor), "r"(oinv), "r"(o));
  bor = nb;
  return q;
#else
  const uint32_t x = t - bor;
  const uint32_t b1 = (t < bor) ? 1u : 0u;
  const uint32_t q = x * oinv;
#ifdef __CUDA_ARCH__
  bor = __umulhi(q, o) + b1;
#else
  bor = (uint32_t)(((uint64_t)q * o) >> 32) + b1;
#endif
  return q;
#endif
}
// limb of (x >> r) given consecutive limbs lo = x[i], hi = x[i+1], 0 < r < 32
TG_HD TG_INLINE uint32_t tg_shr_limb(uint32_t lo, uint32_t hi, int r) {
#ifdef __CUDA_ARCH__
  return __funnelshift_r(lo, hi, r);
#else
  return (lo >> r) | (hi << (32 - r));
#endif
}
// limb i of (x >> r) given lo = x[i], hi = x[i+1], 0 <= r < 32 (r = 0: lo)
TG_HD TG_INLINE uint32_t tg_shr_limb_or_delay(uint32_t lo, uint32_t hi, int r) {
#ifdef __CUDA_ARCH__
  return __funnelshift_r(lo, hi, r);
#else
  return r ? ((lo >> r) | (hi << (32 - r))) : lo;
#endif
}
// limb of (x << r) given lo = x[i-1], hi = x[i], 0 < r < 32
TG_HD TG_INLINE uint32_t tg_shl_limb(uint32_t lo, uint32_t hi, int r) {
#ifdef __CUDA_ARCH__
  return __funnelshift_l(lo, hi, r);
#else
  return (hi << r) | (lo >> (32 - r));
#endif
}
#endif
"""


# ------------------------------------------------- long-vector op tables
#
# The long-vector executor (csrc/longvec.cuh) runs a program as a sequence of
# limb-parallel launches, one per op  dst = ((sum_i m_i * (src_i << s_i)) / o) >> shr,
# each op computed modulo 2^(32 W) over whole vectors (W = slot width).  The
# tables below give, per point set: the evaluation ops (one per point,
# U(p:q) = sum_k p^k q^(n-k) u_k; PAPER.md:16-24 with homogeneous points) and
# the interpolation ops (temps assigned to a minimal set of vector slots by
# liveness), with the per-op look-ahead ("lag") the right shifts need.

LONG_DIGIT = 40          # big multipliers are split into signed 40-bit digits


def _split_mult(m, s):
    """m * 2^s as a list of (digit, shift) with |digit| < 2^(LONG_DIGIT-1)+1."""
    if abs(m) < (1 << 62) // 64:
        return [(m, s)]
    out = []
    sh = s
    while m != 0:
        d = m & ((1 << LONG_DIGIT) - 1)
        if d >= 1 << (LONG_DIGIT - 1):
            d -= 1 << LONG_DIGIT
        out.append((d, sh))
        m = (m - d) >> LONG_DIGIT
        sh += LONG_DIGIT
    return [(d, x) for d, x in out if d != 0]


def long_program(prog: Program, outputs_are_slots=True):
    """Assign slots; returns dict(ops=[(dst, [(src, m, s)], odiv, shr)], outputs, nslots, lag).
    src >= 0: slot, src < 0: input -(k+1).  dst >= 0 slot."""
    inputs = {v: -(k + 1) for k, v in enumerate(prog.inputs)}
    ops = _live_ops(prog, prog.outputs)
    last = {}
    for i, op in enumerate(ops):
        for t in op.terms:
            last[t.var] = i
    for v in prog.outputs:
        last[v] = len(ops)
    where = dict(inputs)
    free, nslots = [], 0
    out_ops = []
    for i, op in enumerate(ops):
        if free:
            free.sort()
            d = free.pop(0)
        else:
            d = nslots
            nslots += 1
        terms = []
        for t in op.terms:
            if t.var == "ZERO":
                continue
            for m, s in _split_mult(t.m, t.s):
                terms.append((where[t.var], m, s))
        out_ops.append((d, terms, op.odiv, op.shr))
        where[op.dst] = d
        for t in op.terms:
            if t.var != "ZERO" and last.get(t.var) == i and where[t.var] >= 0 and t.var not in prog.outputs:
                if where[t.var] not in free:
                    free.append(where[t.var])
    # deficits (limbs of look-ahead consumed below the slot width)
    deficit = {}
    slot_def = {}
    for d, terms, o, shr in out_ops:
        a, r = divmod(shr, 32)
        lag = a + (1 if r else 0)
        dd = 0
        for src, m, s in terms:
            if src >= 0:
                dd = max(dd, slot_def[src] - s // 32)
        slot_def[d] = max(0, dd) + lag
    lag = max([slot_def[where[v]] for v in prog.outputs if where[v] >= 0] + [0])
    outs = [where[v] for v in prog.outputs]
    # sanity: exact execution on random ints through the slot machine
    return dict(ops=out_ops, outputs=outs, nslots=nslots, lag=lag)


def run_long(lp, inputs):
    slots = {}
    def val(src):
        return inputs[-src - 1] if src < 0 else slots[src]
    assert all(d >= 0 for d, _, _, _ in lp["ops"])
    for d, terms, o, shr in lp["ops"]:
        x = sum(m * (val(src) << s) for src, m, s in terms)
        assert x % (o << shr) == 0
        slots[d] = x // (o << shr)
    return [val(s) for s in lp["outputs"]]


def long_eval_program(ps: PointSet):
    """One op per point (direct homogeneous evaluation)."""
    n = ps.n
    ops = []
    for k, (p, q) in enumerate(ps.points):
        terms = []
        for j in range(ps.B):
            c = p**j * q ** (n - j)
            if c:
                sh = (abs(c) & -abs(c)).bit_length() - 1     # powers of two become shifts
                terms += [(-(j + 1), m, s) for m, s in _split_mult(c >> sh, sh)]
        ops.append((k, terms, 1, 0))
    return dict(ops=ops, outputs=list(range(len(ps.points))), nslots=len(ps.points), lag=0)


def long_interp_program(ps: PointSet):
    if ps.B <= 4:
        # PAPER.md:162 matrix form: one op per coefficient, composed from the
        # even-odd + listing program (per_output_programs)
        it = build_interp(ps)
        progs = per_output_programs(it, f"li_{ps.name}")
        ops, outs, ns = [], [], 0
        for j, p in enumerate(progs):
            if not p.ops:
                outs.append(-(it.inputs.index(p.outputs[0]) + 1))
                continue
            op = p.ops[0]
            ops.append((ns, [(-(it.inputs.index(t.var) + 1), t.m, t.s) for t in op.terms], op.odiv, op.shr))
            outs.append(ns)
            ns += 1
        lag = max([((op[3] // 32) + (1 if op[3] % 32 else 0)) for op in ops] + [0])
        return dict(ops=ops, outputs=outs, nslots=ns, lag=lag)
    return long_program(fuse_single_use(build_interp(ps)))


def _growth_S(ps: PointSet):
    return max(sum(abs(p**k * q ** (ps.n - k)) for k in range(ps.B)) for p, q in ps.points)


def emit_long_tables(ps: PointSet) -> str:
    rng = random.Random(7)
    ev = long_eval_program(ps)
    it = long_interp_program(ps)
    # round trip on exact integers through the slot machines
    for _ in range(3):
        U = [rng.randrange(-(1 << 200), 1 << 200) for _ in range(ps.B)]
        V = [rng.randrange(-(1 << 200), 1 << 200) for _ in range(ps.B)]
        EU, EV = run_long(ev, U), run_long(ev, V)
        W = run_long(it, [a * b for a, b in zip(EU, EV)])
        conv = [sum(U[i] * V[k - i] for i in range(ps.B) if 0 <= k - i < ps.B) for k in range(2 * ps.B - 1)]
        assert W == conv, ps.name
    lines = [f"// long-vector tables for {ps.name} (csrc/longvec.cuh)"]
    nm = ps.name
    S = _growth_S(ps)
    lines.append(f"constexpr unsigned long long tg_growthS_{nm} = {S if S < (1 << 64) else 0}ull;")
    # limbs an evaluated operand grows by: e = b + ceil((bitlen(S) + 1) / 32)
    lines.append(f"constexpr int tg_growthLimbs_{nm} = {(S.bit_length() + 1 + 31) // 32};")
    if ps.B <= 4:
        # combined interpolation + recomposition over the common denominator
        # (PAPER.md:162 matrix form, Eq. 1.3): Dc w = sum_j 2^(32 b j) sum_k A'_jk y_k
        it0 = build_interp(ps)
        rows = per_output_programs(it0, f"lc_{nm}")
        NP = ps.npoints
        A, Ds = [], []
        for pr in rows:
            coef = [0] * NP
            if pr.ops:
                op = pr.ops[0]
                for t in op.terms:
                    coef[pr.inputs.index(t.var)] += t.m << t.s
                D = op.odiv << op.shr
            else:
                coef[pr.inputs.index(pr.outputs[0])] = 1
                D = 1
            A.append(coef)
            Ds.append(D)
        Dc = reduce(_lcm, Ds, 1)
        sc = (Dc & -Dc).bit_length() - 1
        lines.append(f"static const long long tg_lcomb_{nm}[{NP}][{NP}] = {{" +
                     ", ".join("{" + ", ".join(str(A[j][k] * (Dc // Ds[j])) for k in range(NP)) + "}" for j in range(NP)) + "};")
        lines.append(f"constexpr unsigned tg_lcombO_{nm} = {Dc >> sc}u;")
        lines.append(f"constexpr int tg_lcombS_{nm} = {sc};")
        # per-row form w_j = (sum_k A_jk y_k) / (o_j 2^s_j) (multi-output interpolation)
        lines.append(f"static const long long tg_lrowA_{nm}[{NP}][{NP}] = {{" +
                     ", ".join("{" + ", ".join(str(A[j][k]) for k in range(NP)) + "}" for j in range(NP)) + "};")
        ro = [D >> ((D & -D).bit_length() - 1) for D in Ds]
        rs = [(D & -D).bit_length() - 1 for D in Ds]
        lines.append(f"static const unsigned tg_lrowO_{nm}[{NP}] = {{" + ", ".join(f"{x}u" for x in ro) + "};")
        lines.append(f"static const int tg_lrowS_{nm}[{NP}] = {{" + ", ".join(str(x) for x in rs) + "};")
    for tag, lp in (("eval", ev), ("interp", it)):
        terms, ops = [], []
        for d, ts, o, shr in lp["ops"]:
            t0 = len(terms)
            for src, m, s in ts:
                terms.append(f"{{{src}, {s}, {m}ll}}")
            sm = sum(abs(m) for _, m, _ in ts)
            wide = 1 if sm >= (1 << 30) else 0
            assert sm < (1 << 61), (nm, tag, sm)
            inv = pow(o, -1, 1 << 32) if o > 1 else 1
            ops.append(f"{{{d}, {t0}, {len(ts)}, {o}u, 0x{inv:08X}u, {shr}, {wide}}}")
        lines.append(f"static const tg_lterm tg_lt_{nm}_{tag}[] = {{" + ", ".join(terms) + "};")
        lines.append(f"static const tg_lop tg_lo_{nm}_{tag}[] = {{" + ", ".join(ops) + "};")
        lines.append(f"static const int tg_lout_{nm}_{tag}[] = {{" + ", ".join(str(x) for x in lp["outputs"]) + "};")
        lines.append(f"constexpr int tg_lnops_{nm}_{tag} = {len(ops)};")
        lines.append(f"constexpr int tg_lnslots_{nm}_{tag} = {lp['nslots']};")
        lines.append(f"constexpr int tg_llag_{nm}_{tag} = {lp['lag']};")
    return "\n".join(lines)


def emit_bigrow_tables(ps: PointSet) -> str:
    """Per-coefficient rows of a point set whose row denominators exceed one
    word (the paper's Toom-8 points): w_j = (sum_k m_jk y_k) / (2^s_j o1_j o2_j)
    with word-sized odd factors o1, o2 (PAPER.md:162 matrix form composed from
    the even-odd + listing program; exactness checked by Program.add)."""
    it = build_interp(ps)
    env = input_forms(it)
    NP = ps.npoints
    M, O1, O2, S = [], [], [], []
    for j, v in enumerate(it.outputs):
        f = env[v]
        D = 1
        for c in f.values():
            D = _lcm(D, c.denominator)
        row = [0] * NP
        for k, c in f.items():
            row[it.inputs.index(k)] = int(c * D)
        s = (D & -D).bit_length() - 1
        o = D >> s
        fs = _word_factors(o) if o > 1 else [1]
        assert len(fs) <= 2, (ps.name, j, fs)
        fs = fs + [1] * (2 - len(fs))
        assert sum(abs(m) for m in row) < (1 << 62)
        M.append(row)
        O1.append(fs[0])
        O2.append(fs[1])
        S.append(s)
        # exactness of the composed row on the symbolic forms
        tot = [0] * it.nunk
        for k, m in enumerate(row):
            fk = it.forms[it.inputs[k]]
            for u in range(it.nunk):
                tot[u] += m * fk[u]
        assert all(x % D == 0 for x in tot) and [x // D for x in tot] == it.forms[v]
    nm = ps.name
    L = [f"// per-coefficient rows of {nm} (k_interp_rows_big)"]
    L.append(f"TG_CONST long long tg_brow_m_{nm}[{NP}][{NP}] = {{" +
             ", ".join("{" + ", ".join(f"{x}ll" for x in r) + "}" for r in M) + "};")
    L.append(f"TG_CONST unsigned tg_brow_o1_{nm}[{NP}] = {{" + ", ".join(f"{x}u" for x in O1) + "};")
    L.append(f"TG_CONST unsigned tg_brow_o2_{nm}[{NP}] = {{" + ", ".join(f"{x}u" for x in O2) + "};")
    L.append(f"TG_CONST unsigned tg_brow_i1_{nm}[{NP}] = {{" + ", ".join(f"0x{_inv32(x):08X}u" for x in O1) + "};")
    L.append(f"TG_CONST unsigned tg_brow_i2_{nm}[{NP}] = {{" + ", ".join(f"0x{_inv32(x):08X}u" for x in O2) + "};")
    L.append(f"TG_CONST int tg_brow_s_{nm}[{NP}] = {{" + ", ".join(str(x) for x in S) + "};")
    L.append(f"constexpr int tg_brow_maxs_{nm} = {max(S)};")
    # the same multipliers as compile-time constants (k_interp_rows_p8s: one
    # IMAD.WIDE.U32 per 27-bit part of |m| into sign-separated 64-bit sums;
    # with limbs below 2^32 every such sum stays below 2^61)
    SPLIT = 27
    for r in M[1:]:
        for sg in (1, -1):
            lo = sum((abs(m) & ((1 << SPLIT) - 1)) for m in r if m * sg > 0) * 0xFFFFFFFF
            hi = sum((abs(m) >> SPLIT) for m in r if m * sg > 0) * 0xFFFFFFFF
            assert lo < (1 << 61) and hi < (1 << 61), (nm, r)
    L.append(f"constexpr int tg_brow_split_{nm} = {SPLIT};")
    L.append(f"TG_HD constexpr long long tg_brow_cx_{nm}(int j, int k) {{")
    L.append(f"  switch (j * {NP} + k) {{")
    for j, r in enumerate(M):
        for k, m in enumerate(r):
            if m:
                L.append(f"    case {j * NP + k}: return {m}ll;")
    L.append("    default: return 0ll;")
    L.append("  }")
    L.append("}")
    return "\n".join(L)


LONG_HEADER = """
// one term m * (src << s) of a long-vector op; src >= 0 slot, src < 0 input -(k+1)
struct tg_lterm { int src; int s; long long m; };
// dst = ((sum of terms) / odiv) >> shr   (odiv odd, oinv = odiv^-1 mod 2^32)
struct tg_lop { int dst; int t0; int nt; unsigned odiv; unsigned oinv; int shr; int wide; };
"""



# ------------------------------------------- matrix-form Toom-16 interpolation
#
# SURVEY §8(f)1 / PAPER.md:162 ("inverting this matrix ... for specific n this
# may be faster"): after the even-odd split (Eqs. 4.5-4.6) the 31-point
# interpolation is two dense solves, done here once symbolically:
#   E_i = y(+p_i/q_i) + y(-p_i/q_i) = 2 sum_{j even} w_j p_i^j q_i^(30-j)
#   O_i = y(+p_i/q_i) - y(-p_i/q_i) = 2 sum_{j odd}  w_j p_i^j q_i^(30-j)
#   w_0 = y_0, w_30 = y_inf;  even rows w_j = (sum_i a_ji E_i + b_j y_0 + c_j y_inf) / D_j
#   y' = y(2:5) - sum_{j even} w_j 2^j 5^(30-j)   (the unpaired point)
#   odd rows  w_j = (sum_i a'_ji O_i + d_j y') / D'_j
# Every D_j = 2^s o_1 o_2 o_3 with coprime odd word factors (primes <= 29);
# every numerator exactly divisible (the selfcheck below runs the pipeline).
# Multipliers (<= 120 bits) are balanced 32-bit digits m = sum_d a_d 2^(32 d).

F1_ND = 4


def _solve_rows(M):
    N = len(M)
    A = [list(map(Fraction, row)) + [Fraction(int(i == r)) for i in range(N)] for r, row in enumerate(M)]
    for c in range(N):
        piv = next(r for r in range(c, N) if A[r][c] != 0)
        A[c], A[piv] = A[piv], A[c]
        inv = 1 / A[c][c]
        A[c] = [x * inv for x in A[c]]
        for r in range(N):
            if r != c and A[r][c] != 0:
                f = A[r][c]
                A[r] = [x - f * y for x, y in zip(A[r], A[c])]
    return [row[N:] for row in A]


def _digits(m, nd=F1_ND):
    """balanced base-2^32 digits, |a_d| <= 2^31"""
    out = []
    for _ in range(nd):
        d = m & 0xFFFFFFFF
        if d >= 1 << 31:
            d -= 1 << 32
        out.append(d)
        m = (m - d) >> 32
    assert m == 0, "multiplier too wide"
    return out


def _word_factor_coprime(o):
    """odd o -> coprime word factors (prime powers packed greedily below 2^32)"""
    f = {}
    p = 3
    while o > 1:
        while o % p == 0:
            f[p] = f.get(p, 0) + 1
            o //= p
        p += 2
    words = []
    for x in sorted([p**e for p, e in f.items()], reverse=True):
        assert x < (1 << 32)
        for i in range(len(words)):
            if words[i] * x < (1 << 32):
                words[i] *= x
                break
        else:
            words.append(x)
    return words


def t16_matrix_form(ps=None):
    ps = ps or pointset_T16_31()
    pts, d = ps.points, 2 * ps.n
    pairs, used = [], set()
    for i, (p, q) in enumerate(pts):
        if p > 0 and q > 0 and (-p, q) in pts:
            j = pts.index((-p, q))
            pairs.append((i, j, p, q))
            used |= {i, j}
    i0, iinf = pts.index((0, 1)), pts.index((1, 0))
    unp = [i for i in range(len(pts)) if i not in used and i not in (i0, iinf)]
    assert len(unp) == 1
    iu = unp[0]
    pu, qu = pts[iu]
    lcm = lambda xs: reduce(_lcm, xs, 1)
    ev = list(range(2, d - 1, 2))
    Ie = _solve_rows([[2 * p**j * q**(d - j) for j in ev] for (_, _, p, q) in pairs])
    even = []
    for r, j in enumerate(ev):
        coef = list(Ie[r]) + [Fraction(0), Fraction(0)]
        for i, (_, _, p, q) in enumerate(pairs):
            coef[len(pairs)] -= Ie[r][i] * 2 * q**d
            coef[len(pairs) + 1] -= Ie[r][i] * 2 * p**d
        D = lcm([c.denominator for c in coef])
        even.append((j, [int(c * D) for c in coef], D))
    od = list(range(1, d, 2))
    Io = _solve_rows([[2 * p**j * q**(d - j) for j in od] for (_, _, p, q) in pairs] + [[pu**j * qu**(d - j) for j in od]])
    odd = []
    for r, j in enumerate(od):
        coef = list(Io[r])
        D = lcm([c.denominator for c in coef])
        odd.append((j, [int(c * D) for c in coef], D))
    ymul = [pu**j * qu**(d - j) for j in range(0, d + 1, 2)]
    return dict(pairs=pairs, i0=i0, iinf=iinf, iu=iu, even=even, odd=odd, ymul=ymul, d=d, pts=pts)


def t16_matrix_selfcheck(F, trials=12, bits=400, seed=7):
    rnd = random.Random(seed)
    d, pts = F["d"], F["pts"]
    for _ in range(trials):
        w = [rnd.getrandbits(bits) - (rnd.getrandbits(1) << (bits - 1)) for _ in range(d + 1)]
        y = [sum(w[j] * p**j * q**(d - j) for j in range(d + 1)) for (p, q) in pts]
        E = [y[a] + y[b] for a, b, _, _ in F["pairs"]]
        O = [y[a] - y[b] for a, b, _, _ in F["pairs"]]
        wr = [None] * (d + 1)
        wr[0], wr[d] = y[F["i0"]], y[F["iinf"]]
        for j, cf, D in F["even"]:
            X = sum(c * x for c, x in zip(cf, E + [y[F["i0"]], y[F["iinf"]]]))
            # the executor's order: / o1 >> s, then / o2, / o3 -- each exact
            s = (D & -D).bit_length() - 1
            words = _word_factor_coprime(D >> s) or [1]
            assert X % words[0] == 0 and (X // words[0]) % (1 << s) == 0
            X = (X // words[0]) >> s
            for o in words[1:]:
                assert X % o == 0
                X //= o
            wr[j] = X
        yp = y[F["iu"]] - sum(wr[j] * m for j, m in zip(range(0, d + 1, 2), F["ymul"]))
        for j, cf, D in F["odd"]:
            X = sum(c * x for c, x in zip(cf, O + [yp]))
            s = (D & -D).bit_length() - 1
            words = _word_factor_coprime(D >> s) or [1]
            X = (X // words[0]) >> s
            for o in words[1:]:
                assert X % o == 0
                X //= o
            wr[j] = X
        assert wr == w, "matrix-form T16 interpolation is not exact"
    return True


def emit_t16_matrix_tables() -> str:
    F = t16_matrix_form()
    t16_matrix_selfcheck(F)
    L = ["// ---- matrix-form Toom-16 interpolation (f1; PAPER.md:162, Eqs. 4.5-4.6), generated and",
         "// checked by toomgen.t16_matrix_form / t16_matrix_selfcheck"]
    NPR = len(F["pairs"])
    L.append(f"constexpr int tg_f1_npairs = {NPR};")
    L.append(f"constexpr int tg_f1_nd = {F1_ND};")
    L.append("constexpr int tg_f1_pair[%d][2] = {%s};" % (NPR, ", ".join("{%d, %d}" % (a, b) for a, b, _, _ in F["pairs"])))
    L.append(f"constexpr int tg_f1_i0 = {F['i0']}, tg_f1_iinf = {F['iinf']}, tg_f1_iu = {F['iu']};")

    def rows(name, R, nsrc):
        NW = 3
        L.append(f"constexpr int tg_f1_{name}_n = {len(R)};")
        L.append(f"constexpr int tg_f1_{name}_j[{len(R)}] = {{" + ", ".join(str(j) for j, _, _ in R) + "};")
        L.append(f"constexpr int tg_f1_{name}_a[{len(R)}][{nsrc}][{F1_ND}] = {{")
        for _, cf, _ in R:
            assert len(cf) == nsrc
            L.append("  {" + ", ".join("{" + ", ".join(str(x) for x in _digits(c)) + "}" for c in cf) + "},")
        L.append("};")
        sh, ws = [], []
        for _, _, D in R:
            s = (D & -D).bit_length() - 1
            words = _word_factor_coprime(D >> s)
            assert len(words) <= NW
            sh.append(s)
            ws.append(words + [1] * (NW - len(words)))
        L.append(f"constexpr int tg_f1_{name}_s[{len(R)}] = {{" + ", ".join(str(x) for x in sh) + "};")
        L.append(f"constexpr unsigned tg_f1_{name}_o[{len(R)}][{NW}] = {{" +
                 ", ".join("{" + ", ".join(f"{x}u" for x in w) + "}" for w in ws) + "};")

    rows("even", F["even"], NPR + 2)
    rows("odd", F["odd"], NPR + 1)
    L.append(f"constexpr int tg_f1_ymul[{len(F['ymul'])}][{F1_ND}] = {{" +
             ", ".join("{" + ", ".join(str(x) for x in _digits(m)) + "}" for m in F["ymul"]) + "};")
    return "\n".join(L)

def generate_all():
    # T16 (31 points, C5's top level) runs through the long-vector path, not
    # the streaming emitter (its multipliers exceed one word).
    sets = [pointset_T3(), pointset_T4(), pointset_paper(8)]
    parts = [HEADER]
    meta = {}
    for ps in sets:
        selfcheck(ps, trials=8)
        ev = fuse_single_use(build_eval(ps))
        it = fuse_single_use(build_interp(ps))
        parts.append(f"// ===== point set {ps.name}: B={ps.B}, points {ps.points}")
        parts.append(f"constexpr int {ps.name}_B = {ps.B};")
        parts.append(f"constexpr int {ps.name}_npoints = {ps.npoints};")
        parts.append(emit_stream_function(ev, f"tg_eval_{ps.name}"))
        parts.append(emit_stream_function(it, f"tg_interp_{ps.name}"))
        # the two halves separately (independent, run in parallel)
        d = 2 * ps.n
        ev_idx = [j for j in range(d + 1) if j % 2 == 0]
        od_idx = [j for j in range(d + 1) if j % 2 == 1]
        parts.append(emit_stream_function(it, f"tg_interp_{ps.name}_even", [it.outputs[j] for j in ev_idx], ev_idx))
        parts.append(emit_stream_function(it, f"tg_interp_{ps.name}_odd", [it.outputs[j] for j in od_idx], od_idx))
        if ps.B <= 4:
            # fused bottom-level kernel tables: one point / one coefficient row per warp
            parts.append(emit_row_tables(ps))
            parts.append("#ifdef __CUDACC__")
            parts.append(emit_row_functions(ps))
            parts.append(emit_evalrow_functions(ps))
            parts.append(emit_rowstep_functions(ps))
            parts.append("#endif")
        meta[ps.name] = dict(B=ps.B, points=ps.points, eval=stats(ev), interp=stats(it))
    parts.append(emit_bigrow_tables(pointset_paper(8)))
    parts.append(LONG_HEADER)
    # P32: the paper's own points 0, +-2^j (j < 31) at B = 32 (PAPER.md:208,
    # "64-bit ... allows B = 32"): divisors up to 2^60 run as
    # 2-adic divisions by their 32-bit word factors on 32-bit limbs
    for ps in [pointset_T3(), pointset_T4(), pointset_paper(8), pointset_T16_31(), pointset_paper(32)]:
        parts.append(emit_long_tables(ps))
    parts.append(emit_t16_matrix_tables())
    return "\n\n".join(parts) + "\n", meta


if __name__ == "__main__":
    import json
    import os
    import sys
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "csrc", "generated", "toom_programs.cuh")
    code, meta = generate_all()
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        f.write(code)
    print(json.dumps(meta, indent=1))

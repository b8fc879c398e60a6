"""Emit csrc/models_gen.cuh: one compile-time topology struct per entry of
paper_2604_09993_b200.topology.COMPILED plus the dispatch table.

Run by __graft_entry__.build() / build.py before nvcc.
"""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2604_09993_b200.topology import COMPILED, key_from_parts  # noqa: E402


def chain(name, vals, default=-1):
    body = " : ".join(f"i == {i} ? {v}" for i, v in enumerate(vals))
    expr = f"{body} : {default}" if vals else str(default)
    return f"  __host__ __device__ static constexpr int {name}(int i) {{ return {expr}; }}\n"


def chol_order(joints):
    """Minimum-degree elimination order of the joint Gram matrix (2x2 blocks;
    joints couple iff they share a link) and the block pattern of its Cholesky
    factor in that order.  Trees eliminated leaves-first have no fill."""
    nj = len(joints)
    links = [set(l for l in (p, c) if l >= 0) for p, c, _ in joints]
    g = {j: {k for k in range(nj) if k != j and links[j] & links[k]} for j in range(nj)}
    remaining = set(range(nj))
    order = []
    depth = {j: 0 for j in range(nj)}  # elimination-tree depth: prefer shallow -> short dependency chain
    while remaining:
        j = min(remaining, key=lambda x: (len(g[x] & remaining), depth[x], x))
        order.append(j)
        nb = g[j] & remaining - {j}
        for a in nb:
            g[a] |= nb - {a}
            depth[a] = max(depth[a], depth[j] + 1)
        remaining.remove(j)
    pos = {j: i for i, j in enumerate(order)}
    lnz = {(i, i) for i in range(nj)}
    for j in range(nj):
        for k in g[j]:
            a, b = pos[j], pos[k]
            if a > b:
                lnz.add((a, b))
    return order, lnz


def chol_code(nj, lnz):
    """Straight-line block LDL^T factorisation + solves of the 2 nj x 2 nj joint Gram
    matrix in elimination order, 2x2 blocks (one joint = one block; only structurally
    nonzero blocks, constant indices only, so every value lives in a register).
    G = L D L^T with unit block-lower L:
        D_b  = G_bb - sum_k W_bk L_bk^T          W_rb = G_rb - sum_k W_rk L_bk^T
        L_rb = W_rb D_b^-1                      (D_b^-1 by the 2x2 adjugate / det)
    one reciprocal per joint on the dependency chain instead of two square roots
    (the chain of the tree's deepest path sets the latency of the primal stage).
    Packed storage LI(r, c) = r (r + 1) / 2 + c: the off-diagonal blocks hold L_rb,
    the diagonal block slots hold D_b^-1 (symmetric: (2b,2b), (2b+1,2b), (2b+1,2b+1));
    Li is not used by the block form (written as 0)."""
    LI = lambda r, c: r * (r + 1) // 2 + c  # noqa: E731
    blk = lambda a, b: (a, b) in lnz  # noqa: E731
    f = ["  __device__ __forceinline__ static void chol_solve(double* L, double* y, double* Li) {\n"]
    for r in range(2 * nj):
        f.append(f"    Li[{r}] = 0.0;\n")
    for b in range(nj):
        ks = [k for k in range(b) if blk(b, k)]
        f.append(f"    double D{b}_00 = L[{LI(2 * b, 2 * b)}], D{b}_10 = L[{LI(2 * b + 1, 2 * b)}], "
                 f"D{b}_11 = L[{LI(2 * b + 1, 2 * b + 1)}];\n")
        for k in ks:  # D -= W_bk L_bk^T (symmetric: lower triangle)
            f.append(f"    D{b}_00 -= W{b}_{k}_00 * L{b}_{k}_00 + W{b}_{k}_01 * L{b}_{k}_01;"
                     f" D{b}_10 -= W{b}_{k}_10 * L{b}_{k}_00 + W{b}_{k}_11 * L{b}_{k}_01;"
                     f" D{b}_11 -= W{b}_{k}_10 * L{b}_{k}_10 + W{b}_{k}_11 * L{b}_{k}_11;\n")
        f.append(f"    const double id{b} = 1.0 / (D{b}_00 * D{b}_11 - D{b}_10 * D{b}_10);\n")
        f.append(f"    const double I{b}_00 = D{b}_11 * id{b}, I{b}_10 = -D{b}_10 * id{b}, I{b}_11 = D{b}_00 * id{b};\n")
        f.append(f"    L[{LI(2 * b, 2 * b)}] = I{b}_00; L[{LI(2 * b + 1, 2 * b)}] = I{b}_10; "
                 f"L[{LI(2 * b + 1, 2 * b + 1)}] = I{b}_11;\n")
        for r in range(b + 1, nj):
            if not blk(r, b):
                continue
            f.append(f"    double W{r}_{b}_00 = L[{LI(2 * r, 2 * b)}], W{r}_{b}_01 = L[{LI(2 * r, 2 * b + 1)}], "
                     f"W{r}_{b}_10 = L[{LI(2 * r + 1, 2 * b)}], W{r}_{b}_11 = L[{LI(2 * r + 1, 2 * b + 1)}];\n")
            for k in ks:
                if not blk(r, k):
                    continue
                for i in range(2):
                    for j in range(2):  # (W_rk L_bk^T)_ij = sum_m W_rk[i][m] L_bk[j][m]
                        f.append(f"    W{r}_{b}_{i}{j} -= W{r}_{k}_{i}0 * L{b}_{k}_{j}0 + W{r}_{k}_{i}1 * L{b}_{k}_{j}1;\n")
            for i in range(2):
                for j in range(2):  # L_rb = W_rb D_b^-1 (D^-1 symmetric: [[I00, I10], [I10, I11]])
                    d0 = f"I{b}_00" if j == 0 else f"I{b}_10"
                    d1 = f"I{b}_10" if j == 0 else f"I{b}_11"
                    f.append(f"    const double L{r}_{b}_{i}{j} = W{r}_{b}_{i}0 * {d0} + W{r}_{b}_{i}1 * {d1};"
                             f" L[{LI(2 * r + i, 2 * b + j)}] = L{r}_{b}_{i}{j};\n")
    solve = []
    for b in range(nj):  # forward: z_b = y_b - sum_k L_bk z_k
        for i in range(2):
            terms = "".join(f" - L[{LI(2 * b + i, 2 * k)}] * y[{2 * k}] - L[{LI(2 * b + i, 2 * k + 1)}] * y[{2 * k + 1}]"
                            for k in range(b) if blk(b, k))
            if terms:
                solve.append(f"    y[{2 * b + i}] = y[{2 * b + i}]{terms};\n")
    for b in range(nj):  # diagonal: w_b = D_b^-1 z_b
        solve.append(f"    {{ const double z0 = y[{2 * b}], z1 = y[{2 * b + 1}];"
                     f" y[{2 * b}] = L[{LI(2 * b, 2 * b)}] * z0 + L[{LI(2 * b + 1, 2 * b)}] * z1;"
                     f" y[{2 * b + 1}] = L[{LI(2 * b + 1, 2 * b)}] * z0 + L[{LI(2 * b + 1, 2 * b + 1)}] * z1; }}\n")
    for b in range(nj - 1, -1, -1):  # backward: x_b = w_b - sum_r L_rb^T x_r
        for i in range(2):
            terms = "".join(f" - L[{LI(2 * r, 2 * b + i)}] * y[{2 * r}] - L[{LI(2 * r + 1, 2 * b + i)}] * y[{2 * r + 1}]"
                            for r in range(b + 1, nj) if blk(r, b))
            if terms:
                solve.append(f"    y[{2 * b + i}] = y[{2 * b + i}]{terms};\n")
    f += solve
    f.append("  }\n")
    # both triangular solves with a given factor (rate-Jacobian tangents reuse the primal factor)
    f.append("  __device__ __forceinline__ static void tri_solve(const double* L, const double* Li, double* y) {\n")
    f.append("    (void)Li;\n")
    f += solve
    f.append("  }\n")
    return "".join(f)


def joint_fill(joints):
    """Block pattern of the joint Gram matrix in JOINT order (joints coupled iff they
    share a link) and of its Cholesky factor with fill (symbolic elimination in joint
    order) -- K3's factorisation order (csrc/cito_node.cuh)."""
    nj = len(joints)
    g = [[False] * nj for _ in range(nj)]
    for j in range(nj):
        for k in range(nj):
            pj, cj, pk, ck = joints[j][0], joints[j][1], joints[k][0], joints[k][1]
            g[j][k] = j == k or (pj >= 0 and (pj == pk or pj == ck)) or cj == ck or (pk >= 0 and cj == pk)
    lm = [row[:] for row in g]
    for c in range(nj):
        for r in range(c + 1, nj):
            if lm[r][c]:
                for r2 in range(c + 1, r + 1):
                    if lm[r2][c]:
                        lm[r][r2] = lm[r2][r] = True
    return g, lm


def chol_code_llt(nj, lnz):
    """(A/B only, CITO_CHOL=llt) Straight-line scalar sparse Cholesky + both triangular solves of the 2 nj x 2 nj
    joint Gram matrix in elimination order (only structurally nonzero entries,
    constant indices only, so every value lives in a register).  Same operation
    order as the loop form it replaces (left-looking columns, reciprocal pivots
    via rsqrt).  L is the packed lower triangle LI(r, c) = r (r + 1) / 2 + c."""
    n = 2 * nj
    nz = lambda r, c: (r // 2, c // 2) in lnz or (r // 2 == c // 2)  # noqa: E731
    LI = lambda r, c: r * (r + 1) // 2 + c  # noqa: E731
    f = ["  __device__ __forceinline__ static void chol_solve(double* L, double* y, double* Li) {\n"]
    for cc in range(n):
        terms = [k for k in range(cc) if nz(cc, k)]
        f.append(f"    {{ double d = L[{LI(cc, cc)}];")
        for k in terms:
            f.append(f" d -= L[{LI(cc, k)}] * L[{LI(cc, k)}];")
        f.append(f" const double il = rsqrt(d); L[{LI(cc, cc)}] = d * il; Li[{cc}] = il;")
        for r in range(cc + 1, n):
            if not nz(r, cc):
                continue
            f.append(f" {{ double x = L[{LI(r, cc)}];")
            for k in range(cc):
                if nz(r, k) and nz(cc, k):
                    f.append(f" x -= L[{LI(r, k)}] * L[{LI(cc, k)}];")
            f.append(f" L[{LI(r, cc)}] = x * il; }}")
        f.append(" }\n")
    solve = []
    for r in range(n):
        solve.append(f"    {{ double x = y[{r}];")
        for k in range(r):
            if nz(r, k):
                solve.append(f" x -= L[{LI(r, k)}] * y[{k}];")
        solve.append(f" y[{r}] = x * Li[{r}]; }}\n")
    for r in range(n - 1, -1, -1):
        solve.append(f"    {{ double x = y[{r}];")
        for k in range(r + 1, n):
            if nz(k, r):
                solve.append(f" x -= L[{LI(k, r)}] * y[{k}];")
        solve.append(f" y[{r}] = x * Li[{r}]; }}\n")
    f += solve
    f.append("  }\n")
    # both triangular solves with a given factor (rate-Jacobian tangents reuse the primal factor)
    f.append("  __device__ __forceinline__ static void tri_solve(const double* L, const double* Li, double* y) {\n")
    f += solve
    f.append("  }\n")
    return "".join(f)


def dirs_for(nl, contacts, implicit, hb_links):
    nq = 3 * nl
    d = set()
    for l in range(nl):
        d.add(3 * l + 2)
        d.add(nq + 3 * l + 2)
    for l in contacts:
        d.add(3 * l + 1)
        d.add(nq + 3 * l)
        d.add(nq + 3 * l + 1)
        if implicit:
            d.add(3 * l)
    for l in hb_links:
        d.add(3 * l + 1)
    return sorted(d)


def main(out_path, entries=None):
    """Write the topology structs + dispatch table of `entries` (default: the bundled
    set, topology.COMPILED) to out_path."""
    parts = ["// GENERATED by gen_models.py from paper_2604_09993_b200/topology.py -- do not edit\n",
             "#pragma once\n\n"]
    table = []
    for name, nl, joints, contacts, implicit, ngo, jl, hb in (COMPILED if entries is None else entries):
        act_idx = []
        a = 0
        for (_, _, act) in joints:
            act_idx.append(a if act else -1)
            a += 1 if act else 0
        dirs = dirs_for(nl, contacts, implicit, hb)
        nq = 3 * nl
        # coordinates whose velocity-row stage increments must be kept (history):
        # v-rows read by the rate Jacobian, and partners of q-rows it reads
        hist = sorted({d - nq for d in dirs if d >= nq} | {d for d in dirs if d < nq})
        hslot = [hist.index(c) if c in hist else -1 for c in range(nq)]
        # state columns whose tangent ever reaches a rate input ("heavy"); the rest are
        # closed-form: q-column c (q_c unread) stays e_c; v-column c (v_c, q_c unread)
        # keeps dv_c = 1 and accumulates dq_c = sum h (sum_i b_i S)
        dset = set(dirs)
        heavy = [c for c in range(2 * nq)
                 if (c in dset) or (c >= nq and (c - nq) in dset)]
        light = [c for c in range(2 * nq) if c not in heavy]
        pushc = [c for c in range(nq) if c not in hist]
        pslot = [pushc.index(c) if c in pushc else -1 for c in range(nq)]
        # structural dependency of rate row rr (vdot rows 0..nq-1, then Omega rows) on state direction kd
        link_of = lambda d: (d % nq) // 3
        comp_of = lambda d: (d % nq) % 3
        ny = 5 * len(contacts) + ngo
        adep = []
        for rr in range(nq + ny):
            row = []
            for d in dirs:
                if rr < nq:  # vdot: theta/omega of every link; implicit terrain: contact-link positions
                    dep = comp_of(d) == 2 or (implicit and d < nq and link_of(d) in contacts)
                elif rr - nq < 5 * len(contacts):  # Omega rows of contact i: its link's coordinates only
                    dep = link_of(d) == contacts[(rr - nq) // 5]
                else:  # mixed path rows
                    dep = True
                row.append(1 if dep else 0)
            adep.append(row)
        adep_bits = [sum(b << k for k, b in enumerate(row)) for row in adep]
        s = f"struct Topo_{name} {{\n"
        s += (f"  static constexpr int NL = {nl}, NJ = {len(joints)}, NA = {a}, NC = {len(contacts)}, "
              f"NGO = {ngo}, NJL = {len(jl)}, NHB = {len(hb)}, NDIRX = {len(dirs)}, NHIST = {len(hist)}, "
              f"NPUSH = {len(pushc)};\n")
        order, lnz = chol_order(joints)
        blocks = sorted(lnz)
        s += f"  static constexpr int NBLK = {len(blocks)};\n"
        s += chain("blk_a", [a for a, _ in blocks])
        s += chain("blk_b", [b for _, b in blocks])
        s += chain("jperm", order)
        lbits = [sum(1 << b for b in range(len(joints)) if (a, b) in lnz) for a in range(len(joints))]
        s += ("  __host__ __device__ static constexpr bool lnzb(int a, int b) { return (("
              + "".join(f"a == {i} ? {v}u : " for i, v in enumerate(lbits)) + "0u) >> b) & 1u; }\n")
        if joints:
            s += (chol_code_llt if os.environ.get("CITO_CHOL") == "llt" else chol_code)(len(joints), lnz)
        jg, jl_ = joint_fill(joints)
        for nm, mat in (("jfill_g", jg), ("jfill_l", jl_)):
            bits = [sum(1 << b for b in range(len(joints)) if mat[a][b]) for a in range(len(joints))]
            s += (f"  __host__ __device__ static constexpr bool {nm}(int a, int b) {{ return (("
                  + "".join(f"a == {i} ? {v}u : " for i, v in enumerate(bits)) + "0u) >> b) & 1u; }\n")
        s += f"  static constexpr int NHCOL = {len(heavy)}, NLCOL = {len(light)};\n"
        s += chain("hcol", heavy)
        s += chain("lcol", light)
        s += chain("hslot", hslot)
        s += chain("pslot", pslot)
        s += ("  __host__ __device__ static constexpr bool adep(int rr, int kd) { return (("
              + " : ".join(f"rr == {i} ? {v}ull" for i, v in enumerate(adep_bits)) + " : 0ull) >> kd) & 1ull; }\n")
        s += f"  static constexpr bool IMPLICIT = {'true' if implicit else 'false'};\n"
        s += chain("jparent", [p for p, _, _ in joints])
        s += chain("jchild", [c for _, c, _ in joints])
        s += chain("jact", act_idx)
        s += chain("clink", list(contacts))
        s += chain("jl_joint", list(jl))
        s += chain("hb_link", list(hb))
        s += chain("dir", dirs)
        s += "};\n\n"
        parts.append(s)
        table.append((key_from_parts(nl, joints, contacts, implicit, ngo, jl, hb), name))
    parts.append("#define CITO_FOR_EACH_TOPOLOGY(X) \\\n")
    parts.append(" \\\n".join(f'  X(Topo_{n}, "{k}")' for k, n in table))
    parts.append("\n")
    with open(out_path, "w") as f:
        f.write("".join(parts))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(HERE, "models_gen.cuh"))

"""Generates tests/golden/*.npz — independent golden vectors for the oracle pin.

The reference (Eigen-based C++) cannot be built in this image and has no
tests or fixtures of its own, so the pins are:
  * SPEC.md's [OP] examples (encoded directly in tests/test_oracle_kat.py);
  * these fixtures, computed with numpy / scipy / pure Python restatements
    that share no code with oracle/dmc_oracle.c or libdmcg: dense Laplacian
    from face sets, numpy products, numpy.linalg.eigh, numpy.linalg.lstsq on
    the stacked system [L; S] x = [delta; a] (a QR route, not the normal
    equations), Python float quantiser, bit-at-a-time DMC1 serializer
    (reference src/stream.cpp:172-292, src/quantize.cpp:50-60).

Run: python tests/golden/make_golden.py   (writes small_*.npz next to it)
"""
import os
import struct

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def icosphere(level):
    t = (1 + 5 ** 0.5) / 2
    v = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t), (0, -1, -t),
         (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    v = [np.array(p) / np.linalg.norm(p) for p in v]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
         (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
         (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(level):
        mid = {}

        def m(a, b):
            key = (min(a, b), max(a, b))
            if key not in mid:
                p = (v[a] + v[b]) / 2
                v.append(p / np.linalg.norm(p))
                mid[key] = len(v) - 1
            return mid[key]
        nf = []
        for a, b, c in f:
            ab, bc, ca = m(a, b), m(b, c), m(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        f = nf
    return np.array(v), np.array(f, dtype=np.uint32)


def dense_laplacian(faces, n):
    nb = [set() for _ in range(n)]
    for a, b, c in faces:
        for x, y in ((a, b), (b, c), (c, a)):
            nb[x].add(y)
            nb[y].add(x)
    L = np.zeros((n, n))
    for i in range(n):
        L[i, i] = len(nb[i])
        for j in nb[i]:
            L[i, j] = -1.0
    return L


def widened(lo, hi):
    a = np.float32(lo)
    if float(a) > lo:
        a = np.nextafter(a, np.float32(-np.inf))
    b = np.float32(hi)
    if float(b) < hi:
        b = np.nextafter(b, np.float32(np.inf))
    return a, b


def quantize(mn, mx, bits, x):
    levels = 1 << bits
    if mn == mx:
        return 0
    m = float(mn)
    w = (float(mx) - m) / levels
    t = np.floor((x - m) / w)
    if t <= 0:
        return 0
    if t >= levels - 1:
        return levels - 1
    return int(t)


def stride_anchors(n, n_c):
    idx = sorted(set(j * n // n_c for j in range(n_c)))
    used = set(idx)
    i = 0
    while len(idx) < n_c and i < n:
        if i not in used:
            idx.append(i)
            used.add(i)
        i += 1
    return sorted(idx)


class Bits:
    def __init__(self):
        self.out = bytearray()
        self.pending = 0
        self.fill = 0

    def put(self, v, bits):
        for b in range(bits - 1, -1, -1):
            self.pending = (self.pending << 1) | ((v >> b) & 1)
            self.fill += 1
            if self.fill == 8:
                self.out.append(self.pending & 0xFF)
                self.pending = 0
                self.fill = 0

    def take(self):
        if self.fill:
            self.out.append((self.pending << (8 - self.fill)) & 0xFF)
        return bytes(self.out)


def main():
    rng = np.random.default_rng(20111010)
    verts, faces = icosphere(1)          # 42 vertices, 80 faces
    n, F, k_l, bits = len(verts), 12, 6, 10
    t = np.arange(F)
    axes = []
    for a in range(3):
        w = rng.normal(size=(3, 3))
        traj = verts[:, a:a + 1] * (1 + 0.1 * np.sin(2 * np.pi * t / F)[None, :])
        traj = traj + 0.05 * np.outer(verts @ w[0], np.cos(2 * np.pi * 2 * t / F))
        traj = traj + 0.01 * rng.normal(size=(n, F))
        axes.append(np.ascontiguousarray(traj))
    L = dense_laplacian(faces, n)
    delta = [L @ x for x in axes]
    R = [x.T @ x for x in axes]
    U, ev = [], []
    for r in R:
        w, V = np.linalg.eigh(r)
        w, V = w[::-1], V[:, ::-1].copy()
        for j in range(F):
            i = int(np.argmax(np.abs(V[:, j])))
            if V[i, j] < 0:
                V[:, j] = -V[:, j]
        U.append(V)
        ev.append(w)
    coeffs = [U[a].T @ delta[a].T for a in range(3)]  # F x n
    rmin = np.zeros((3, k_l), np.float32)
    rmax = np.zeros((3, k_l), np.float32)
    q = np.zeros((3, k_l, n), np.uint32)
    for a in range(3):
        for r in range(k_l):
            lo, hi = widened(float(coeffs[a][r].min()), float(coeffs[a][r].max()))
            rmin[a, r], rmax[a, r] = lo, hi
            q[a, r] = [quantize(lo, hi, bits, float(x)) for x in coeffs[a][r]]
    n_c = max(1, min(n, int(round(0.05 * n))))
    idx = np.array(stride_anchors(n, n_c), np.uint32)
    S = np.zeros((n_c, n))
    S[np.arange(n_c), idx] = 1.0
    A = np.vstack([L, S])
    solve = np.stack([np.linalg.lstsq(A, np.vstack([delta[a], axes[a][idx]]), rcond=None)[0]
                      for a in range(3)])
    # dictionary + anchors, then the DMC1 bytes of this encoding
    dict_q = np.zeros((3, F, F), np.uint32)  # [a][col][row]
    for a in range(3):
        for j in range(F):
            dict_q[a, j] = [quantize(np.float32(-1), np.float32(1), 16, float(x)) for x in U[a][:, j]]
    amin = np.zeros(3, np.float32)
    amax = np.zeros(3, np.float32)
    aq = np.zeros((3, n_c, F), np.uint32)
    for a in range(3):
        vals = axes[a][idx]
        amin[a], amax[a] = widened(float(vals.min()), float(vals.max()))
        aq[a] = [[quantize(amin[a], amax[a], 16, float(x)) for x in row] for row in vals]
    out = bytearray(b"DMC1")
    out += struct.pack("<HBBIIHHIIBBBB", 1, 4, 0, n, F, 1, 0, k_l, n_c, 16, 16, 8, 0)
    out += struct.pack("<I", len(faces))
    for f in faces:
        out += struct.pack("<III", *[int(x) for x in f])
    for a in range(3):
        b = Bits()
        for v in dict_q[a].reshape(-1):
            b.put(int(v), 16)
        out += b.take()
        for r in range(k_l):
            out += struct.pack("<ffB", rmin[a, r], rmax[a, r], bits)
        b = Bits()
        for r in range(k_l):
            if rmin[a, r] != rmax[a, r]:
                for v in q[a, r]:
                    b.put(int(v), bits)
        out += b.take()
    for i in idx:
        out += struct.pack("<I", int(i))
    for a in range(3):
        out += struct.pack("<ff", amin[a], amax[a])
        b = Bits()
        for v in aq[a].reshape(-1):
            b.put(int(v), 16)
        out += b.take()
    np.savez_compressed(os.path.join(HERE, "small_ico1.npz"), faces=faces, axes=np.stack(axes),
                        L=L, delta=np.stack(delta), R=np.stack(R), U=np.stack(U), ev=np.stack(ev),
                        coeffs=np.stack(coeffs), k_l=k_l, bits=bits, rmin=rmin, rmax=rmax, q=q,
                        anchor_idx=idx, solve=solve, dict_q=dict_q, anchor_min=amin,
                        anchor_max=amax, anchor_q=aq, stream=np.frombuffer(bytes(out), np.uint8))
    print("wrote small_ico1.npz", n, F, len(out), "bytes stream")


if __name__ == "__main__":
    main()

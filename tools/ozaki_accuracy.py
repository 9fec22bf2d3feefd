"""Accuracy of an Ozaki-style int8 emulation of the FP64 MTTKRP (DESIGN.md
§9.6), emulated exactly on the CPU: the tensor split into S signed int8
digit planes under one global power-of-two exponent, the Khatri-Rao factor
A_f into S planes under one exponent per column, the products of digit
planes with s + t <= S - 1 accumulated exactly (int64 here; int32 on the
tensor cores, which is exact for o-groups up to ~18k) per diagonal, then
combined in FP64 and scaled by the o-rows' product per o-group -- the same
arithmetic the tcgen05 kind::i8 kernel would do.  Prints the relative
Frobenius error against the FP64 MTTKRP for S = 4..8.

    python tools/ozaki_accuracy.py
"""
import numpy as np


def digits(x, e, S):
    """x / 2^e in (-1/2, 1/2] -> S signed digits d_s (|d_0| <= 64, |d_s| <= 64),
    x ~= sum_s d_s 2^(e - 7 (s + 1))."""
    r = x / np.ldexp(1.0, e)
    out = []
    for _ in range(S):
        r = r * 128.0
        d = np.rint(r)
        out.append(d.astype(np.int64))
        r = r - d
    return out


def mttkrp_mode2_ozaki(y, a0, a1, S):
    """G[i2, r] = sum_{i1} a1[i1, r] sum_{i0} y[i0, i1, i2] a0[i0, r] (y first-mode-fastest,
    stored as y[i2, i1, i0] in C order)."""
    i2n, i1n, i0n = y.shape
    ey = int(np.ceil(np.log2(np.abs(y).max()))) + 1
    ea = np.ceil(np.log2(np.abs(a0).max(axis=0))).astype(int) + 1  # per column
    yd = digits(y, ey, S)
    ad = [np.stack([digits(a0[:, r], ea[r], S)[s] for r in range(a0.shape[1])], axis=1) for s in range(S)]
    g = np.zeros((i2n, a0.shape[1]))
    for o in range(i1n):  # one o-group: exact integer products per diagonal, then FP64
        acc = [np.zeros((i2n, a0.shape[1]), dtype=np.int64) for _ in range(S)]
        for s in range(S):
            for t in range(S - s):
                acc[s + t] += yd[s][:, o, :] @ ad[t]
        val = np.zeros((i2n, a0.shape[1]))
        for dd in range(S - 1, -1, -1):  # smallest terms first
            val += acc[dd].astype(np.float64) * np.ldexp(1.0, -7 * dd)
        g += a1[o][None, :] * (val * np.ldexp(1.0, ey - 14) * np.ldexp(np.ones(a0.shape[1]), ea)[None, :])
    return g


def main():
    rng = np.random.Generator(np.random.Philox(3))
    shape, r = (64, 48, 128), 40  # (I2, I1, I0), rank
    cases = {
        "uniform [0,1) (the bench data)": (rng.random(shape), rng.random((shape[2], r)), rng.random((shape[1], r))),
        "normal": (rng.standard_normal(shape), rng.standard_normal((shape[2], r)), rng.standard_normal((shape[1], r))),
        "lognormal, sigma 3 (wide dynamic range)": (rng.lognormal(0, 3, shape) * rng.choice([-1, 1], shape),
                                                    rng.lognormal(0, 3, (shape[2], r)), rng.random((shape[1], r))),
    }
    for name, (y, a0, a1) in cases.items():
        ref = np.einsum("kji,ir,jr->kr", y, a0, a1)
        errs = []
        for S in range(4, 9):
            g = mttkrp_mode2_ozaki(y, a0, a1, S)
            errs.append(f"S={S}: {np.linalg.norm(g - ref) / np.linalg.norm(ref):.2e}")
        print(f"{name}: " + ", ".join(errs))


if __name__ == "__main__":
    main()

"""numpy emulation of param_grads_kernel's chain (geometry.cu project_core + backward_projection_core)
in a chosen dtype, to find the step where float32 loses the parameter gradients of one primitive."""
import numpy as np


def chain(T, raw, cam, psi, sg, dilation=0.3):
    f = lambda x: np.asarray(x, dtype=T)
    out = {}
    mu = f(raw[0:3]); s = np.exp(f(raw[3:6])).astype(T); q = f(raw[6:10])
    fx, fy = f(cam[0]), f(cam[1])
    W = f(cam[6:18]).reshape(3, 4)
    t = (W[:, :3] @ mu + W[:, 3]).astype(T)
    n = np.sqrt((q * q).sum(dtype=T)).astype(T)
    w, x, y, z = (q / n).astype(T)
    two = T(2)
    R = f([[1 - two * (y * y + z * z), two * (x * y - w * z), two * (x * z + w * y)],
           [two * (x * y + w * z), 1 - two * (x * x + z * z), two * (y * z - w * x)],
           [two * (x * z - w * y), two * (y * z + w * x), 1 - two * (x * x + y * y)]])
    M = (R * s[None, :]).astype(T)
    sigma = (M @ M.T).astype(T)
    zc = t[2]
    J = f([[fx / zc, 0, -fx * t[0] / (zc * zc)], [0, fy / zc, -fy * t[1] / (zc * zc)]])
    Tj = (J @ W[:, :3]).astype(T)
    raw2 = (Tj @ sigma @ Tj.T).astype(T)
    cov = f([psi * raw2[0, 0] + dilation, psi * T(0.5) * (raw2[0, 1] + raw2[1, 0]), psi * raw2[1, 1] + dilation])
    a, b, c = cov
    inv = T(1) / (a * c - b * b)
    ca, cb, cc = c * inv, -b * inv, a * inv
    ga, gb, gc = f(sg[4]), T(0.5) * f(sg[5]), f(sg[6])
    C = f([[ca, cb], [cb, cc]]); G = f([[ga, gb], [gb, gc]])
    dcov = (-(C @ G @ C)).astype(T)
    gmu2 = f(sg[7:9])
    out.update(t=t, sigma=sigma, Tj=Tj, cov=cov, conic=f([ca, cb, cc]), dcov=dcov)
    gxy = T(0.5) * (dcov[0, 1] + dcov[1, 0])
    graw = f([[psi * dcov[0, 0], psi * gxy], [psi * gxy, psi * dcov[1, 1]]])
    gt = (graw @ Tj).astype(T)              # 2x3
    d_sigma = (Tj.T @ gt).astype(T)         # 3x3
    d_tj = (two * (gt @ sigma)).astype(T)   # 2x3
    d_j = (d_tj @ W[:, :3].T).astype(T)     # 2x3
    z2, z3 = zc * zc, zc * zc * zc
    d_t = f([d_j[0, 2] * (-fx / z2), d_j[1, 2] * (-fy / z2),
             d_j[0, 0] * (-fx / z2) + d_j[1, 1] * (-fy / z2) + d_j[0, 2] * (two * fx * t[0] / z3) + d_j[1, 2] * (two * fy * t[1] / z3)])
    d_t_cov = d_t.copy()
    d_t = d_t + f([gmu2[0] * fx / zc, gmu2[1] * fy / zc, -gmu2[0] * fx * t[0] / z2 - gmu2[1] * fy * t[1] / z2])
    d_mu = (W[:, :3].T @ d_t).astype(T)
    d_m = ((d_sigma + d_sigma.T) @ M).astype(T)
    d_scale = (R * d_m).sum(axis=0, dtype=T)
    out.update(gt=gt, d_sigma=d_sigma, d_tj=d_tj, d_j=d_j, d_t_cov=d_t_cov, d_t=d_t, d_mu=d_mu, d_m=d_m, d_scale=d_scale * s)
    return out


def compare(raw, cam, psi, sg):
    a = chain(np.float32, raw, cam, psi, sg)
    b = chain(np.float64, raw, cam, psi, sg)
    for key in b:
        den = np.abs(b[key]).max()
        print(f"{key:8s} max|f32-f64|/max|f64| = {np.abs(a[key] - b[key]).max() / max(den, 1e-300):.2e}   f64 = {np.array2string(np.asarray(b[key]).ravel(), precision=4, max_line_width=200)}")

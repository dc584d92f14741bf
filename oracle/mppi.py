"""TEST INFRASTRUCTURE ONLY — oracle of the MPPI controller on the batched step
(§V, Eq. (14)-(15); SPEC mppi module
S:393-457).  Plain fp64 numpy; shares no code with the CUDA path.

  noise      eps[k] = sigma sqrt(-2 ln(1 - u1)) cos(2 pi u2), u1, u2 the top 24
             bits of SplitMix64(seed + 2k), SplitMix64(seed + 2k + 1) over 2^24,
             k = ((iteration P + p) N + i) H Q + t Q + j (the counter-based
             generator both sides implement; integers bit-exact)
  samples    U_i = clip(U_bar + eps_i, lo, hi)           ("clip actions")
  control    incremental position control: command += u_t, then the
             joint PD torque tau = kp (command - q) - kd qdot  (reading R27)
  cost       Eq. (15): c(x) = w1 (1 - (q_t . q_obj)^2) + w2 |p_x - t_x| + w3 |p_y - t_y|
             + w4 |p_z - t_z| + w5 sum_i |p_obj - p_tip_i|^2 + w6 |q_robot - q_ref|^2
             + Omega [p_z < z_fallen];  V(x) = phi1 |p_obj - p_t|^2 + phi2 (1 - (q_t . q_obj)^2)
             J_i = sum_{t=0}^{H-1} c(x_t) + V(x_H)   (Eq. (14))
  update     w_i = exp(-(J_i - min J)/lambda) / sum, U_bar <- clip(sum_i w_i U_i, lo, hi)
             (min subtraction, normalised weights); a non-finite J_i
             (diverged rollout) counts as +inf, weight 0, and a problem with no
             finite J keeps its plan (reading R29; the paper is silent)
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def uniform24(x: int) -> float:
    return (splitmix64(x) >> 40) / float(1 << 24)


def noise(seed, iteration, P, N, H, Q, sigma):
    """eps (P, N, H, Q)."""
    out = np.zeros((P, N, H, Q))
    for p in range(P):
        for i in range(N):
            for t in range(H):
                for j in range(Q):
                    k = (((iteration * P + p) * N + i) * H + t) * Q + j
                    u1 = uniform24((seed + 2 * k) & M64)
                    u2 = uniform24((seed + 2 * k + 1) & M64)
                    out[p, i, t, j] = sigma * np.sqrt(-2.0 * np.log(1.0 - u1)) * np.cos(2.0 * np.pi * u2)
    return out


def samples(plan, eps, lo, hi):
    """plan (P, H, Q), eps (P, N, H, Q) -> U (P, N, H, Q)."""
    return np.clip(plan[:, None] + eps, lo, hi)


def pd_torque(command, q, qd, kp, kd):
    return kp * (command - q) - kd * qd


def cost(task, p_obj, q_obj, tips, q_robot, problem, terminal: bool):
    """Eq. (15) for one world: running cost c(x) or terminal V(x)."""
    pt = np.asarray(task["target_pos"][problem], float)
    qt = np.asarray(task["target_quat"][problem], float)
    qo = np.asarray(q_obj, float) / np.linalg.norm(q_obj)
    cq = 1.0 - float(qt @ qo) ** 2
    if terminal:
        return task["phi1"] * float(np.sum((p_obj - pt) ** 2)) + task["phi2"] * cq
    w = task["w"]
    c = w[0] * cq + w[1] * abs(p_obj[0] - pt[0]) + w[2] * abs(p_obj[1] - pt[1]) + w[3] * abs(p_obj[2] - pt[2])
    c += w[4] * sum(float(np.sum((p_obj - tp) ** 2)) for tp in tips)
    c += w[5] * float(np.sum((q_robot - np.asarray(task["q_ref"], float)) ** 2))
    c += task["omega_fallen"] * (1.0 if p_obj[2] < task["z_fallen"] else 0.0)
    return c


def update(J, U, lam, lo, hi, plan_prev=None):
    """J (P, N), U (P, N, H, Q) -> new plan (P, H, Q), weights (P, N)."""
    P, N, H, Q = U.shape
    plan = np.zeros((P, H, Q)) if plan_prev is None else np.array(plan_prev, np.float64)
    w = np.zeros((P, N))
    for p in range(P):
        Jp = np.where(np.isfinite(J[p]), J[p], np.inf)     # reading R29
        if not np.isfinite(Jp).any():
            continue                                        # keep the previous plan, weights 0
        e = np.where(np.isfinite(Jp), np.exp(-(Jp - Jp.min()) / lam), 0.0)
        w[p] = e / e.sum()
        plan[p] = np.clip(np.einsum("n,nhq->hq", w[p], U[p]), lo, hi)
    return plan, w

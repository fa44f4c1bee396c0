"""The paper's analytic cost model (§3, Eq. 2-10; Table 2 at P:376-398)
-- TEST INFRASTRUCTURE ONLY.  It pins the model shapes the build uses (e.g. the
70B FFN width F = 28672 that Table 2 implies), the steady-state batch composition
of Eq. 2 and the compute-bound optimum of Eq. 9 that
bench.py reports against, to the numbers the paper prints
(tests/golden/table2_llama2_70b_8xa100.json, optimal_throughput.json).

Per-operation accounting follows SURVEY.md Appendix A (the paper gives the
formulas only in aggregate):
  dense GEMM [B, K] x [K, N] per layer: FLOP 2 B N K, bytes (N K + B K + B N) * 2;
  decode attention: E = n_dec * (p + d/2) * 2 Hkv hd L elements of K/V read,
    FLOP 2 E R_GQA, bytes 2 E + the q and o rows (2 n_dec D * 2 L);
  prefill attention: 4 (B_req / (d+1)) p^2 D L FLOP (non-causal count);
  communication (P:340-346 with Table 2's (N-1) factor, App. B item 4):
    4 B D * 2 bytes * L * (N - 1) over the aggregate one-way NVLink bandwidth.
"""
from __future__ import annotations

from typing import Dict


def steady_state(b_dense: float, p: int, d: int):
    """Eq. 2: B_dense = B_req (p + d) / (d + 1); returns (B_req, n_prefill_req, n_decode)."""
    b_req = b_dense * (d + 1) / (p + d)
    return b_req, b_req / (d + 1), b_req * d / (d + 1)


def table2(D: int, L: int, Hq: int, Hkv: int, hd: int, F: int, b_dense: int, p: int, d: int, n_gpu: int,
           flops_per_gpu: float, mem_bw_per_gpu: float, net_bw_per_gpu: float, dtype_bytes: int = 2
           ) -> Dict[str, Dict[str, float]]:
    """Rows of Table 2: compute (GFLOP), memory (GB), network (GB), T_compute / T_mem / T_net (ms)."""
    B = b_dense
    flops, mem_bw, net_bw = flops_per_gpu * n_gpu, mem_bw_per_gpu * n_gpu, net_bw_per_gpu * n_gpu
    rows = {}

    def gemm(name, N, K):
        f = 2.0 * B * N * K * L
        m = (N * K + B * K + B * N) * dtype_bytes * L
        rows[name] = {"compute": f / 1e9, "memory": m / 1e9, "network": 0.0,
                      "t_compute": f / flops * 1e3, "t_mem": m / mem_bw * 1e3, "t_net": 0.0}

    gemm("GEMM-KQV", (Hq + 2 * Hkv) * hd, D)
    gemm("GEMM-O", D, Hq * hd)
    gemm("GEMM-UG", 2 * F, D)
    gemm("GEMM-D", D, F)
    b_req, n_pre, n_dec = steady_state(B, p, d)
    R = Hq // Hkv
    E = n_dec * (p + d / 2) * 2 * Hkv * hd * L           # K/V elements read per step
    f = 2.0 * E * R
    m = E * dtype_bytes + 2 * n_dec * D * dtype_bytes * L
    rows["Decode Attention"] = {"compute": f / 1e9, "memory": m / 1e9, "network": 0.0,
                                "t_compute": f / flops * 1e3, "t_mem": m / mem_bw * 1e3, "t_net": 0.0}
    f = 4.0 * n_pre * p * p * D * L
    rows["Prefill Attention"] = {"compute": f / 1e9, "t_compute": f / flops * 1e3}
    net = 4.0 * B * D * dtype_bytes * L * (n_gpu - 1)
    rows["Communication"] = {"network": net / 1e9, "memory": net / 1e9, "t_net": net / net_bw * 1e3,
                             "t_mem": net / mem_bw * 1e3}
    rows["Total"] = {"t_compute": sum(r.get("t_compute", 0.0) for r in rows.values())}
    return rows


def optimal_throughput(compute_flops: float, p_model: float) -> float:
    """Eq. 9: tokens/s = Compute / (2 P_model)."""
    return compute_flops / (2.0 * p_model)

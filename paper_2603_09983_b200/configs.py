"""The five BASELINE.json workload shapes.

d / ffn / layer counts / shared experts come from the public model configs,
not from the reference (which has no FFN at all; its "expert" is
expert_bytes = 25 MB, core/src/config.cpp:27). Gate normalisation per model:
Mixtral and Qwen3 renormalise over the top-k (Eq. 3, gate_mode 0);
Qwen1.5-MoE and DeepSeek-V2-Lite take the softmax over all N (gate_mode 1).
Shared experts are expressed as units of d_ffn rows (Qwen1.5: one 5632-row
shared expert = 4 units of 1408; DeepSeek-V2-Lite: 2 x 1408 = 2 units).
Qwen1.5-MoE scales its shared expert per token by sigmoid(w_sg . h_t)
(`shared_expert_gate`, shared_gate=1); DeepSeek-V2-Lite adds its shared
experts with weight 1.
DeepSeek-V2-Lite's first layer is dense in the real model; BASELINE.json
names 27 layers and all 27 are modeled as MoE layers here (one layer more of
expert work than the model has).
"""
from __future__ import annotations

from dataclasses import dataclass, replace


# Synthetic weight scale: bf16 ~ N(0, SYNTH_STD^2) for every gate/up/down
# entry. The layers have no norms, so the residual stream h_{l+1} = h_l + y_l
# must not blow up over 24-48 layers: a SwiGLU expert scales as |h|^2, and at
# std 0.02 the Mixtral shape (d = 4096, ffn = 14336) overflows to inf by
# layer ~16. At 0.006 every BASELINE shape keeps |y| << |h| (values stay
# finite and parity-checkable; timing does not depend on the values).
SYNTH_STD = 0.006


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    n_layers: int
    n_experts: int
    top_k: int
    gamma: int
    d_model: int
    d_ffn: int
    n_shared_units: int = 0
    gate_mode: int = 0
    cache_ratio: float = 0.17
    description: str = ""
    shared_gate: int = 0  # MOESPAC_SHARED_GATE_*: 1 = per-token sigmoid(w_sg . h) (Qwen1.5-MoE)

    @property
    def tokens(self) -> int:
        return self.gamma + 1

    @property
    def expert_bytes(self) -> int:
        return 3 * self.d_model * self.d_ffn * 2

    def with_(self, **kw) -> "WorkloadConfig":
        return replace(self, **kw)

    def model_desc(self, ffn_kernel: int = 0, parallel_mode: int = 0):
        from . import abi
        return abi.ModelDesc(self.n_layers, self.n_experts, self.top_k, self.gamma, self.d_model, self.d_ffn,
                             self.n_shared_units, self.gate_mode, ffn_kernel, parallel_mode, self.shared_gate)


CONFIGS = {
    "tiny": WorkloadConfig("tiny", 1, 8, 2, 4, 512, 1024, 0, 0, 0.17,
                           "tiny synthetic MoE layer: 8 experts top-2, d=512, ffn=1024, draft_len=4"),
    "mixtral": WorkloadConfig("mixtral", 32, 8, 2, 4, 4096, 14336, 0, 0, 1.0,
                              "Mixtral-8x7B-shaped MoE layer: 8 experts top-2, d=4096, ffn=14336, draft_len=4, bf16"),
    "qwen15": WorkloadConfig("qwen15", 24, 60, 4, 6, 2048, 1408, 4, 1, 0.5,
                             "Qwen1.5-MoE-A2.7B shape: 60 experts top-4 + shared expert, draft_len=6, 50% cache",
                             shared_gate=1),
    "dsv2": WorkloadConfig("dsv2", 27, 64, 6, 8, 2048, 1408, 2, 1, 0.17,
                           "DeepSeek-V2-Lite shape: 64 routed experts top-6, 27 layers, draft_len=8"),
    "qwen3": WorkloadConfig("qwen3", 48, 128, 8, 8, 2048, 768, 0, 0, 0.17,
                            "Qwen3-30B-A3B shape: 128 experts top-8, cache-budget sweep 10-100%"),
}


# HWB hardware profile (HardwareProfile, core/include/moesim/workload_balancer.hpp:15-21)
# calibrated to one B200 box of this pool instead of the reference's defaults
# (core/src/config.cpp:23-27: t_cpu 100 us per token-activation, t_gpu 40 us
# per expert pass, t_io 400 us per expert load, t_draft 300 us per token,
# expert_bytes 25 MB). Rates measured in round 2 (profiles/bench_r2*):
#   host cold path, 16 threads, AVX-512 BF16 over the pinned arena: 90 GB/s
#     (Qwen3 @ 0.17: 136 missed experts x 9.44 MB in 14.2 ms per step)
#   K3 on HBM: ~5 TB/s per resident expert pass (0.7-0.94 of the copy peak)
#   pinned host -> HBM expert loads: 48 GB/s (46-53 measured)
#   draft phase: 2e9-parameter bf16 stand-in at 6.99 TB/s per token
# t_cpu is charged per token-activation by the reference; a miss with one
# token costs a whole expert read on the host, so one expert read it is.
B200_RATES = {"host_cold_Bps": 90e9, "k3_Bps": 5e12, "h2d_Bps": 48e9, "draft_s_per_token": 4e9 / 6.99e12}


def b200_hwb_profile(w: WorkloadConfig) -> dict:
    """SchedConfig profile fields for workload w on B200 (see B200_RATES)."""
    eb = w.expert_bytes
    r = B200_RATES
    return {"t_cpu_unit_ns": round(eb / r["host_cold_Bps"] * 1e9), "t_gpu_unit_ns": round(eb / r["k3_Bps"] * 1e9),
            "t_io_unit_ns": round(eb / r["h2d_Bps"] * 1e9), "t_draft_unit_ns": round(r["draft_s_per_token"] * 1e9),
            "expert_bytes": eb}


HWB_PROFILES = {"reference": lambda w: {}, "b200": b200_hwb_profile}


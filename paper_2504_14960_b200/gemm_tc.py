"""tcgen05/TMEM/TMA grouped GEMM (bf16 in, fp32 accumulate) -- placeholder
until the sm_100a kernel lands; `available()` gates its use."""


def available() -> bool:
    return False


def supports(**kw) -> bool:
    return False


def fused_act_ok(pk) -> bool:
    return False

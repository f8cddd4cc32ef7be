"""Attention shapes used by the attention tools: (q_lens, kv_lens, hq, hkv, hd, mode)."""
CASES = {
    "c2": ([400] * 35, [700] * 35, 32, 32, 128, True),
    "qwen": ([1024] * 8, [8192] * 8, 28, 4, 128, True),
    "vit80": ([29640], [29640], 16, 16, 80, False),
    "win80": ([29640], [29640], 16, 16, 80, "win"),
}

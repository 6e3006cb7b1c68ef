"""A/B helper for the tools: variant strings in the old env-style spelling
("HEP_FFN_PAIR=0 HEP_ST256=1") applied through the library's explicit tuning API
(hep_tuning_set; the library itself never reads the environment)."""

from __future__ import annotations

NAMES = {
    "HEP_ST256": "st256", "HEP_PAIR_WAIT_CLUSTER": "pair_wait_cluster", "HEP_FFN_PAIR": "ffn_pair",
    "HEP_FFN_LIGHT_ROWS": "ffn_light_rows", "HEP_WGRAD_ORDER": "wgrad_order", "HEP_L2POL": "l2_policy",
    "HEP_LIGHT_FIRST": "light_first", "HEP_RASTER_GM1": "raster_gm1", "HEP_RASTER_GM2": "raster_gm2",
    "HEP_SCHED_LEXMIN_WARPS": "sched_lexmin_warps", "HEP_LSU256": "lsu256", "HEP_FFN_CLOCK": "ffn_clock",
    "HEP_ROUTER_TILE_ROWS": "router_tile_rows", "HEP_WAVE_SYNC": "pair_wave_sync", "HEP_LP_DSM": "lp_dsm", "HEP_LIGHT_WAVE_SYNC": "light_wave_sync",
    "HEP_ROUTER_MC": "router_mc", "HEP_ROUTER_PAIR": "router_pair", "HEP_WGRAD_WAVE_SYNC": "wgrad_wave_sync", "HEP_WGRAD_RASTER": "wgrad_raster",
    "HEP_SCHED_ROUTE_SERIAL": "sched_route_serial",
}


def parse(variant: str) -> dict:
    """'HEP_FFN_PAIR=0 st256=1' -> {'ffn_pair': 0, 'st256': 1} (either spelling)."""
    out = {}
    for kv in variant.split():
        k, _, v = kv.partition("=")
        if k == "HEP_RASTER_GM":
            out["raster_gm1"] = out["raster_gm2"] = int(v)
            continue
        out[NAMES.get(k, k)] = int(v)
    return out


def apply(variant: str, base: dict | None = None) -> dict:
    """Reset to ``base`` (the tuning saved before the A/B) and apply ``variant``."""
    from paper_2511_16947_b200 import _lib

    if base is not None:
        _lib.set_tuning(**base)
    fields = parse(variant)
    if fields:
        _lib.set_tuning(**fields)
    return fields

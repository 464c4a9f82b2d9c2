"""CPU float64 oracle — TEST INFRASTRUCTURE ONLY (see aurora_oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Shares no code with the CUDA path.
"""
from .aurora_oracle import (ACCEPT, DISCARD, PAD, bf16_bits_to_f64, target_scan, target_scan_topk, verify,
                            row_targets, loss_fwd, loss_bwd, loss_bwd_sampled, dlogits_rows, step, step_topk, step_variants, warmup_lr, adamw_step)

__all__ = ["ACCEPT", "DISCARD", "PAD", "bf16_bits_to_f64", "target_scan", "target_scan_topk", "verify", "row_targets",
           "loss_fwd", "loss_bwd", "loss_bwd_sampled", "dlogits_rows", "step", "step_topk", "step_variants", "warmup_lr", "adamw_step"]

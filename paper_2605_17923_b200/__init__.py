"""B200-native (sm_100a) rebuild of AdaptiveLoad's accelerator hot path (arxiv 2605.17923).

Mirrors the reference package ``adaptiveload`` (/root/reference/pkg/src/adaptiveload) for the
hot path only:

* ``adaln``     -- fused LayerNorm-Modulate operator (CUDA kernels behind a C ABI)
* ``shapes``    -- latent sequence-length arithmetic and bucket catalogs
* ``scheduler`` -- dual-constraint / equal-token batch-size policies
* ``sampler``   -- per-rank weighted bucket draws (bit-exact with the reference) and the
                   imbalance metrics
* ``dp_step``   -- synthetic Wan-style DiT-block data-parallel step (NCCL all-reduce)
* ``errors``    -- the reference's exception hierarchy
"""

__version__ = "0.1.0"

"""CPU oracles -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import anything here, and only as the checker
or as the timed CPU baseline -- never as the product path.  The product
(`paper_2309_16669_b200`) never imports this package and fails loudly when
its CUDA library is missing.

Modules:
  transform_oracle  numpy float64 restatement of crop -> hflip -> antialiased
                    bilinear -> normalize (K1).  Pinned: boxes are the
                    reference sampler's own output (tests/golden); index rule
                    and weights are checked against torch's antialiased
                    bilinear; libswscale (the reference's scaler) is
                    cross-checked when a copy is loadable.
  vit_oracle        torch fp32 restatement of the ViT video encoder, blockwise
                    attention and CLIP InfoNCE from PAPER.md.  The reference has
                    no encoder/attention/loss code or tests, so
                    there is no reference output to pin against; instead
                    tests/test_vit_oracle_pins.py pins it to independent public
                    formulations: scaled_dot_product_attention, nn.Conv3d tubelet
                    embedding, TransformerEncoderLayer(norm_first) and open_clip's
                    ClipLoss formula.
  swscale_ref       libswscale (the reference's own scaler) via ctypes, called as
                    codec.cpp:226-246 does: the augment workload's reference arm.
  cpu_baseline      timed CPU restatement of K1 (the `port` baseline).
"""

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
                    attention and CLIP InfoNCE from PAPER.md.  PARITY UNPINNED:
                    the reference has no encoder/attention/loss code or tests
                    (SURVEY.md 8(c)); these follow the paper text only.
"""

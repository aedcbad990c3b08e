# round-2 pass 34: first staged-row variant (per-store predicates inside a
# runtime branch: 870 M warp instructions, slower) — superseded by pass 35.

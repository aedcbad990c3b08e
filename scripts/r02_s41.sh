# round-2 pass 41: first f32 fixed-tap 4:3 consumer, three STG.128 per lane
# plane row straight to global memory (1.69 ms at c2: 347 M partial L2 sector
# writes) — superseded by pass 42's warp-staged plane rows.

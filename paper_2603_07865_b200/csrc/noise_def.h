// K4's noise generator, shared by the device kernels (align.cu) and the C restatement
// (oracle/semwarm_oracle.c). Philox4x32 with 7 rounds: the fewest rounds for which Salmon et al.
// (SC'11, "Parallel random numbers: as easy as 1, 2, 3") report the 4x32 Philox passing all of
// TestU01's BigCrush; Random123's default of 10 adds a safety margin. On B200 each round's two
// 32x32->64 products issue on the quarter-rate IMAD.WIDE path, and with 10 rounds the generator
// alone took about the HBM time of the align + noise pass (K4).
#pragma once
#define SW_PHILOX_ROUNDS 7

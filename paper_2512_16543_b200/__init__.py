"""B200-native RZF precoder update (WB-arSVD), drop-in for the leorzf L1 core."""

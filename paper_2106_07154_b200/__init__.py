"""B200-native LTS3 / TRiSK shallow-water path (drop-in for the reference mswm)."""

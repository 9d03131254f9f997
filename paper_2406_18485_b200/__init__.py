"""B200-native (sm_100a) 2D-Attention: head-parallel all-to-all x Double-Ring
context-parallel attention behind the reference's operator API."""

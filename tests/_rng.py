"""SplitMix64 stream identical to seasim::detail::Rng (common.hpp:41-74):
next_u64 (:46-51), next_double (:54), next_below (:70).  Used to replay the
reference's seeded property test (kv_cache_test.cpp:124-181) op for op."""
M64 = (1 << 64) - 1


class Rng:
    def __init__(self, seed: int):
        self.state = seed & M64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def next_below(self, bound: int) -> int:
        return self.next_u64() % bound

// urg_sim_part.cu -- one slice [URG_PART_LO, URG_PART_HI) of the kernel instantiation rows
// (compiled once per slice with -DURG_PART_LO/-DURG_PART_HI/-DURG_PART_FN; see build.py).
#include "urg_sim.cuh"

template <int R, bool IN>
struct PartRow {
    static const void *get(uint32_t) { return nullptr; }
};
template <int R>
struct PartRow<R, true> {
    static const void *get(uint32_t col) { return UrgRow<R>::get(col); }
};

#define URG_ROW(r) \
    case r: return PartRow<r, (URG_PART_LO <= r && r < URG_PART_HI)>::get(col);

const void *URG_PART_FN(uint32_t row, uint32_t col)
{
    switch (row) {
        URG_ROW(0) URG_ROW(1) URG_ROW(2) URG_ROW(3) URG_ROW(4) URG_ROW(5) URG_ROW(6) URG_ROW(7) URG_ROW(8)
        URG_ROW(9) URG_ROW(10) URG_ROW(11) URG_ROW(12) URG_ROW(13) URG_ROW(14) URG_ROW(15) URG_ROW(16)
        URG_ROW(17) URG_ROW(18) URG_ROW(19) URG_ROW(20) URG_ROW(21) URG_ROW(22) URG_ROW(23) URG_ROW(24)
        URG_ROW(25) URG_ROW(26) URG_ROW(27) URG_ROW(28) URG_ROW(29) URG_ROW(30) URG_ROW(31) URG_ROW(32)
        URG_ROW(33) URG_ROW(34) URG_ROW(35) URG_ROW(36) URG_ROW(37)
    default: return nullptr;
    }
}

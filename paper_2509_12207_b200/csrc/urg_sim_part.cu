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
        URG_ROW(17)
    default: return nullptr;
    }
}

// Degree dispatch to the per-n translation units.
#include "dg_internal.h"

namespace dg {

#define DG_DECL(n)                                            \
    int upload_tables_n##n(const HostTables&);                \
    cudaError_t launch_cell_n##n(const KParams&, cudaStream_t); \
    cudaError_t launch_gen_n##n(const KParams&, cudaStream_t);  \
    int cell_info_n##n(LaunchInfo*);                          \
    int gen_info_n##n(LaunchInfo*);
DG_DECL(2) DG_DECL(3) DG_DECL(4) DG_DECL(5) DG_DECL(6) DG_DECL(7) DG_DECL(8) DG_DECL(9) DG_DECL(10) DG_DECL(11)

#define DG_CASES(call)                                                                                  \
    switch (k + 1) {                                                                                    \
    case 2: return call(2); case 3: return call(3); case 4: return call(4); case 5: return call(5);     \
    case 6: return call(6); case 7: return call(7); case 8: return call(8); case 9: return call(9);     \
    case 10: return call(10); case 11: return call(11);                                                 \
    default: break;                                                                                     \
    }

int upload_tables(int k, const HostTables& t)
{
#define DG_UP(n) upload_tables_n##n(t)
    DG_CASES(DG_UP)
    return -1;
}

cudaError_t launch_cell(int k, const KParams& p, cudaStream_t s)
{
#define DG_LA(n) launch_cell_n##n(p, s)
    DG_CASES(DG_LA)
    return cudaErrorInvalidValue;
}

cudaError_t launch_gen(int k, const KParams& p, cudaStream_t s)
{
#define DG_LG(n) launch_gen_n##n(p, s)
    DG_CASES(DG_LG)
    return cudaErrorInvalidValue;
}

int gen_launch_info(int k, LaunchInfo* info)
{
#define DG_GI(n) gen_info_n##n(info)
    DG_CASES(DG_GI)
    return -1;
}

int cell_launch_info(int k, LaunchInfo* info)
{
#define DG_IN(n) cell_info_n##n(info)
    DG_CASES(DG_IN)
    return -1;
}

}  // namespace dg

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

namespace dg {

#define DG_VDECL(n, m)                                                    \
    int upload_tables_vb_n##n##_m##m(const HostTables&);                  \
    cudaError_t launch_vb_n##n##_m##m(const KParams&, cudaStream_t);      \
    int vb_info_n##n##_m##m(LaunchInfo*);
#define DG_VPAIR(n, m2) DG_VDECL(n, n) DG_VDECL(n, m2)
DG_VPAIR(2, 4) DG_VPAIR(3, 5) DG_VPAIR(4, 6) DG_VPAIR(5, 7) DG_VPAIR(6, 8) DG_VPAIR(7, 9) DG_VPAIR(8, 10) DG_VPAIR(9, 11)

#define DG_VCASES(call)                                                                            \
    switch ((k + 1) * 100 + m) {                                                                   \
    case 202: return call(2, 2); case 204: return call(2, 4); case 303: return call(3, 3);         \
    case 305: return call(3, 5); case 404: return call(4, 4); case 406: return call(4, 6);         \
    case 505: return call(5, 5); case 507: return call(5, 7); case 606: return call(6, 6);         \
    case 608: return call(6, 8); case 707: return call(7, 7); case 709: return call(7, 9);         \
    case 808: return call(8, 8); case 810: return call(8, 10); case 909: return call(9, 9);        \
    case 911: return call(9, 11);                                                                  \
    default: break;                                                                                \
    }

bool vb_available(int k, int m) { return k >= 1 && k <= 8 && (m == k + 1 || m == k + 3); }

int upload_tables_vb(int k, int m, const HostTables& t)
{
#define DG_VU(n, mm) upload_tables_vb_n##n##_m##mm(t)
    DG_VCASES(DG_VU)
    return -1;
}

cudaError_t launch_vb(int k, int m, const KParams& p, cudaStream_t s)
{
#define DG_VL(n, mm) launch_vb_n##n##_m##mm(p, s)
    DG_VCASES(DG_VL)
    return cudaErrorInvalidValue;
}

int vb_launch_info(int k, int m, LaunchInfo* info)
{
#define DG_VI(n, mm) vb_info_n##n##_m##mm(info)
    DG_VCASES(DG_VI)
    return -1;
}

}  // namespace dg

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
// (n, m) pairs of the variable-velocity kernel: m = n (q = 2p), n + 2 (q = 2p + 4, the paper's
// Taylor-Green run) and ceil((3k + 5) / 2) (q = 3p + 4) while m <= 16
DG_VDECL(2, 2)
DG_VDECL(2, 4)
DG_VDECL(3, 3)
DG_VDECL(3, 5)
DG_VDECL(3, 6)
DG_VDECL(4, 4)
DG_VDECL(4, 6)
DG_VDECL(4, 7)
DG_VDECL(5, 5)
DG_VDECL(5, 7)
DG_VDECL(5, 9)
DG_VDECL(6, 6)
DG_VDECL(6, 8)
DG_VDECL(6, 10)
DG_VDECL(7, 7)
DG_VDECL(7, 9)
DG_VDECL(7, 12)
DG_VDECL(8, 8)
DG_VDECL(8, 10)
DG_VDECL(8, 13)
DG_VDECL(9, 9)
DG_VDECL(9, 11)
DG_VDECL(9, 15)
DG_VDECL(10, 10)
DG_VDECL(10, 12)
DG_VDECL(10, 16)
DG_VDECL(11, 11)
DG_VDECL(11, 13)

#define DG_VCASES(call)                 \
    switch ((k + 1) * 100 + m) {        \
    case 202: return call(2, 2); case 204: return call(2, 4); case 303: return call(3, 3); case 305: return call(3, 5); case 306: return call(3, 6); case 404: return call(4, 4); case 406: return call(4, 6); case 407: return call(4, 7); case 505: return call(5, 5); case 507: return call(5, 7); case 509: return call(5, 9); case 606: return call(6, 6); case 608: return call(6, 8); case 610: return call(6, 10); case 707: return call(7, 7); case 709: return call(7, 9); case 712: return call(7, 12); case 808: return call(8, 8); case 810: return call(8, 10); case 813: return call(8, 13); case 909: return call(9, 9); case 911: return call(9, 11); case 915: return call(9, 15); case 1010: return call(10, 10); case 1012: return call(10, 12); case 1016: return call(10, 16); case 1111: return call(11, 11); case 1113: return call(11, 13); \
    default: break;                     \
    }

bool vb_available(int k, int m)
{
    switch ((k + 1) * 100 + m) {
    case 202: case 204: case 303: case 305: case 306: case 404: case 406: case 407: case 505: case 507: case 509: case 606: case 608: case 610: case 707: case 709: case 712: case 808: case 810: case 813: case 909: case 911: case 915: case 1010: case 1012: case 1016: case 1111: case 1113: return true;
    default: return false;
    }
}

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

namespace dg {

// (n, m) pairs of the multilinear-geometry kernel (dg_geo.cuh): m = n (q = 2p), n + 2 (q = 2p + 4) and
// ceil((3k + 5) / 2) (Problem C's q = 3p + 4) while the cell's shared memory fits
// (m <= 16)
#define DG_GDECL(n, m)                                                    \
    int upload_tables_geo_n##n##_m##m(const HostTables&);                 \
    cudaError_t launch_geo_n##n##_m##m(const KParams&, cudaStream_t);     \
    int geo_info_n##n##_m##m(LaunchInfo*);
DG_GDECL(2, 2)
DG_GDECL(2, 4)
DG_GDECL(3, 3)
DG_GDECL(3, 5)
DG_GDECL(3, 6)
DG_GDECL(4, 4)
DG_GDECL(4, 6)
DG_GDECL(4, 7)
DG_GDECL(5, 5)
DG_GDECL(5, 7)
DG_GDECL(5, 9)
DG_GDECL(6, 6)
DG_GDECL(6, 8)
DG_GDECL(6, 10)
DG_GDECL(7, 7)
DG_GDECL(7, 9)
DG_GDECL(7, 12)
DG_GDECL(8, 8)
DG_GDECL(8, 10)
DG_GDECL(8, 13)
DG_GDECL(9, 9)
DG_GDECL(9, 11)
DG_GDECL(9, 15)
DG_GDECL(10, 10)
DG_GDECL(10, 12)
DG_GDECL(10, 16)
DG_GDECL(11, 11)
DG_GDECL(11, 13)

#define DG_GCASES(call)                 \
    switch ((k + 1) * 100 + m) {        \
    case 202: return call(2, 2); case 204: return call(2, 4); case 303: return call(3, 3); case 305: return call(3, 5); case 306: return call(3, 6); case 404: return call(4, 4); case 406: return call(4, 6); case 407: return call(4, 7); case 505: return call(5, 5); case 507: return call(5, 7); case 509: return call(5, 9); case 606: return call(6, 6); case 608: return call(6, 8); case 610: return call(6, 10); case 707: return call(7, 7); case 709: return call(7, 9); case 712: return call(7, 12); case 808: return call(8, 8); case 810: return call(8, 10); case 813: return call(8, 13); case 909: return call(9, 9); case 911: return call(9, 11); case 915: return call(9, 15); case 1010: return call(10, 10); case 1012: return call(10, 12); case 1016: return call(10, 16); case 1111: return call(11, 11); case 1113: return call(11, 13); \
    default: break;                     \
    }

bool geo_available(int k, int m)
{
    switch ((k + 1) * 100 + m) {
    case 202: return true; case 204: return true; case 303: return true; case 305: return true; case 306: return true; case 404: return true; case 406: return true; case 407: return true; case 505: return true; case 507: return true; case 509: return true; case 606: return true; case 608: return true; case 610: return true; case 707: return true; case 709: return true; case 712: return true; case 808: return true; case 810: return true; case 813: return true; case 909: return true; case 911: return true; case 915: return true; case 1010: return true; case 1012: return true; case 1016: return true; case 1111: return true; case 1113: return true;
    default: return false;
    }
}

int upload_tables_geo(int k, int m, const HostTables& t)
{
#define DG_GU(n, mm) upload_tables_geo_n##n##_m##mm(t)
    DG_GCASES(DG_GU)
    return -1;
}

cudaError_t launch_geo(int k, int m, const KParams& p, cudaStream_t s)
{
#define DG_GL(n, mm) launch_geo_n##n##_m##mm(p, s)
    DG_GCASES(DG_GL)
    return cudaErrorInvalidValue;
}

int geo_launch_info(int k, int m, LaunchInfo* info)
{
#define DG_GI2(n, mm) geo_info_n##n##_m##mm(info)
    DG_GCASES(DG_GI2)
    return -1;
}

}  // namespace dg

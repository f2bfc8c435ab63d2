// Host build of the engine's crmath.cuh for CPU tests (pinned against mpmath and glibc).
#include "../../paper_2509_21963_b200/csrc/crmath.cuh"
extern "C" {
double crm_log(double x) { return itercur_b200::crm::log_cr(x); }
double crm_cos(double x) { return itercur_b200::crm::cos_cr(x); }
double crm_box_muller(double u1, double u2) { return itercur_b200::crm::box_muller_cos(u1, u2); }
}

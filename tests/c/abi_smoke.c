/* Plain C client of librtgs.so: proves the boundary is a C ABI (no C++ / torch types), and checks
 * the host-side behaviour that needs no GPU: version, status strings, argument validation and the
 * workspace queries.  Built and run by tests/test_c_abi.py. */
#include <stdio.h>
#include <string.h>

#include "rtgs.h"

#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
      return 1;                                               \
    }                                                         \
  } while (0)

int main(void) {
  CHECK(rtgs_version() == 1);
  CHECK(strcmp(rtgs_status_string(RTGS_OK), "RTGS_OK") == 0);
  CHECK(strcmp(rtgs_status_string(RTGS_ERR_WORKSPACE), "RTGS_ERR_WORKSPACE") == 0);
  rtgs_camera cam = {500.f, 500.f, 319.5f, 239.5f, 640, 480};
  rtgs_camera bad = {-1.f, 500.f, 319.5f, 239.5f, 640, 480};
  rtgs_pose pose = {{1, 0, 0, 0, 1, 0, 0, 0, 1}, {0, 0, 0}};
  rtgs_gaussians g;
  memset(&g, 0, sizeof(g));
  g.n = 10;  /* no arrays: rejected */
  g.sh_degree = 3;
  rtgs_projected pr;
  memset(&pr, 0, sizeof(pr));
  CHECK(rtgs_project_gaussians(&g, &pose, &cam, &pr, NULL) == RTGS_ERR_INVALID_ARG);
  g.n = 0;
  CHECK(rtgs_project_gaussians(&g, &pose, &bad, &pr, NULL) == RTGS_ERR_INVALID_ARG);
  rtgs_bins b;
  memset(&b, 0, sizeof(b));
  CHECK(rtgs_bin_and_sort(&pr, 0, &cam, NULL, &b, NULL, 0, NULL) == RTGS_ERR_INVALID_ARG);
  CHECK(rtgs_bin_workspace_size(1000, &cam, 1u << 16) > 0);
  CHECK(rtgs_bin_workspace_size(-1, &cam, 1u << 16) == 0);
  CHECK(rtgs_backward_workspace_size(100) >= 100 * 16 * sizeof(float));
  CHECK(rtgs_classify_workspace_size(&cam) > 0);
  CHECK(rtgs_insert_workspace_size(1000, 64) > 0);
  CHECK(rtgs_icp_workspace_size(&cam, 3) > 0 && rtgs_icp_workspace_size(&cam, 9) == 0);
  CHECK(rtgs_topk_workspace_size(&cam) > 0);
  CHECK(rtgs_bin_cached_workspace_size(100, &cam, 1u << 16) > 0);
  CHECK(rtgs_decode_rgbd(NULL, NULL, 0, 0, 5000.f, NULL, NULL, NULL) == RTGS_OK);
  CHECK(rtgs_decode_rgbd(NULL, NULL, 64, 48, 0.f, NULL, NULL, NULL) == RTGS_ERR_INVALID_ARG);
  rtgs_hparams hp = {1e-3f, 5e-4f, 2.5e-5f, 4e-3f, 1e-3f, 0.9, 0.999, 1e-15};
  rtgs_params prm;
  memset(&prm, 0, sizeof(prm));
  prm.sh_degree = 3;
  CHECK(rtgs_adam_step_unstable(&prm, NULL, 0, NULL, NULL, NULL, NULL, NULL, 0, 1000.f, &hp, 0, NULL, NULL, NULL) ==
        RTGS_ERR_INVALID_ARG); /* step must be >= 1 */
  printf("c abi ok: %llu launches\n", (unsigned long long)rtgs_launch_count());
  return rtgs_launch_count() == 0 ? 0 : 1;
}

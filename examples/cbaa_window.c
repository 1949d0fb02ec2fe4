/* Plain-C user of the CBAA C ABI (include/cbaa.h): no Python, no torch.
 *
 *   cbaa_window <pairs.bin> [theta]
 *
 * pairs.bin holds n little-endian uint32 inner IPs followed by n uint32 outer IPs (SoA, host order).
 * One window: reset -> host-ingest update (the library copies the host arrays to the GPU) -> detect,
 * then the super hosts are printed as "ip estimate" lines, largest estimate first. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "cbaa.h"

int main(int argc, char** argv) {
  if (argc < 2) {
    fprintf(stderr, "usage: %s pairs.bin [theta]\n", argv[0]);
    return 1;
  }
  uint32_t theta = argc > 2 ? (uint32_t)atoi(argv[2]) : 1024;
  FILE* f = fopen(argv[1], "rb");
  if (!f) { perror("open"); return 1; }
  fseek(f, 0, SEEK_END);
  long bytes = ftell(f);
  fseek(f, 0, SEEK_SET);
  uint64_t n = (uint64_t)bytes / 8;
  uint32_t* buf = (uint32_t*)malloc((size_t)bytes + 8);
  if (!buf || fread(buf, 1, (size_t)bytes, f) != (size_t)bytes) { fprintf(stderr, "read failed\n"); return 1; }
  fclose(f);

  cbaa_config cfg;
  cbaa_config_default(&cfg);            /* paper geometry */
  cbaa_handle* h = NULL;
  int rc = cbaa_create(&cfg, 0, &h);
  if (rc) { fprintf(stderr, "cbaa_create: %s\n", cbaa_strerror(rc)); return 2; }
  if ((rc = cbaa_reset(h, NULL)) || (rc = cbaa_update_host(h, buf, buf + n, n, NULL))) {
    fprintf(stderr, "update: %s (%s)\n", cbaa_strerror(rc), cbaa_last_error(h));
    return 2;
  }
  uint64_t cap = 1 << 16, found = 0;
  cbaa_host* out = (cbaa_host*)malloc(cap * sizeof(cbaa_host));
  rc = cbaa_detect(h, theta, out, cap, &found, NULL, NULL);
  if (rc && rc != CBAA_E_TUPLE_CAP) {
    fprintf(stderr, "detect: %s (%s)\n", cbaa_strerror(rc), cbaa_last_error(h));
    return 2;
  }
  printf("# %llu pairs, %llu super hosts (theta = %u)\n", (unsigned long long)n, (unsigned long long)found, theta);
  for (uint64_t k = 0; k < found && k < cap; ++k)
    printf("%u.%u.%u.%u %.3f\n", out[k].ip >> 24, (out[k].ip >> 16) & 255, (out[k].ip >> 8) & 255, out[k].ip & 255,
           out[k].estimate);
  cbaa_destroy(h);
  free(out);
  free(buf);
  return 0;
}

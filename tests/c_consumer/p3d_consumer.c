/* A plain C consumer of libp3d.so (test infrastructure): what a binding in
 * another language links against.  It checks that the header's structs have
 * the library's sizes and ABI version, then runs the host-side design reader
 * (p3d_parse_design: no GPU needed) on a file and prints what it read as one
 * JSON line: counts, scalars and checksums of the CSR arrays, or the error
 * code and message for a malformed design. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "p3d.h"

static char* slurp(const char* path, long* len) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  *len = ftell(f);
  fseek(f, 0, SEEK_SET);
  char* buf = (char*)malloc((size_t)*len + 1);
  if (fread(buf, 1, (size_t)*len, f) != (size_t)*len) { fclose(f); free(buf); return NULL; }
  fclose(f);
  buf[*len] = 0;
  return buf;
}

int main(int argc, char** argv) {
  if (p3d_abi_version() != P3D_ABI_VERSION) { fprintf(stderr, "abi version\n"); return 2; }
  if (p3d_sizeof_topology() != sizeof(p3d_topology) || p3d_sizeof_grid() != sizeof(p3d_grid) ||
      p3d_sizeof_cloud() != sizeof(p3d_cloud) || p3d_sizeof_gp() != sizeof(p3d_gp) ||
      p3d_sizeof_loop_state() != sizeof(p3d_loop_state) ||
      p3d_sizeof_gp2d_ctl() != sizeof(p3d_gp2d_ctl) ||
      p3d_sizeof_gp2d_state() != sizeof(p3d_gp2d_state)) {
    fprintf(stderr, "struct size mismatch between p3d.h and libp3d.so\n");
    return 3;
  }
  if (argc < 2) { printf("{\"abi\": %d}\n", p3d_abi_version()); return 0; }
  long len = 0;
  char* text = slurp(argv[1], &len);
  if (!text) { fprintf(stderr, "cannot read %s\n", argv[1]); return 4; }
  void* h = NULL;
  const int rc = p3d_parse_design(text, (int64_t)len, &h);
  if (rc != P3D_OK) {
    char msg[512];
    p3d_last_error(msg, sizeof msg);
    printf("{\"rc\": %d, \"error\": \"", rc);
    for (const char* c = msg; *c; ++c) {
      if (*c == '"' || *c == '\\') putchar('\\');
      putchar(*c);
    }
    printf("\"}\n");
    free(text);
    return 0;
  }
  int64_t cnt[5];
  double sc[9];
  p3d_parsed_counts(h, cnt, sc);
  const int64_t I = cnt[0], N = cnt[1], P = cnt[2];
  uint8_t* mac = (uint8_t*)malloc((size_t)(I ? I : 1));
  double* wt = (double*)malloc(sizeof(double) * (size_t)(I ? I : 1));
  double* ht = (double*)malloc(sizeof(double) * (size_t)(I ? I : 1));
  double* wb = (double*)malloc(sizeof(double) * (size_t)(I ? I : 1));
  double* hb = (double*)malloc(sizeof(double) * (size_t)(I ? I : 1));
  int64_t* ptr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
  int64_t* pin = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P ? P : 1));
  double* o[4];
  for (int k = 0; k < 4; ++k) o[k] = (double*)malloc(sizeof(double) * (size_t)(P ? P : 1));
  char* in_names = (char*)malloc((size_t)cnt[3] + 1);
  char* net_names = (char*)malloc((size_t)cnt[4] + 1);
  p3d_parsed_fill(h, mac, wt, ht, wb, hb, ptr, pin, o[0], o[1], o[2], o[3], in_names, net_names);
  p3d_parsed_free(h);
  long long sum_ptr = 0, sum_pin = 0, n_macro = 0;
  double sum_size = 0.0, sum_off = 0.0;
  for (int64_t j = 0; j <= N; ++j) sum_ptr += ptr[j];
  for (int64_t p = 0; p < P; ++p) {
    sum_pin += pin[p] * (p % 7 + 1);
    for (int k = 0; k < 4; ++k) sum_off += o[k][p] * (k + 1);
  }
  for (int64_t i = 0; i < I; ++i) {
    n_macro += mac[i] != 0;
    sum_size += wt[i] + 2 * ht[i] + 3 * wb[i] + 4 * hb[i];
  }
  printf("{\"rc\": 0, \"n_inst\": %lld, \"n_net\": %lld, \"n_pin\": %lld, \"n_macro\": %lld, "
         "\"sum_ptr\": %lld, \"sum_pin\": %lld, \"sum_size\": %.17g, \"sum_off\": %.17g, "
         "\"scalars\": [%.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g, %.17g]}\n",
         (long long)I, (long long)N, (long long)P, n_macro, sum_ptr, sum_pin, sum_size, sum_off,
         sc[0], sc[1], sc[2], sc[3], sc[4], sc[5], sc[6], sc[7], sc[8]);
  free(text);
  return 0;
}

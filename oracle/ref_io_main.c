/* ref_io_main.c -- TEST INFRASTRUCTURE ONLY: command-line access to the
 * reference's output formats (vtk.hpp:17-66, through oracle/_ref/libokref.so)
 * from a process without numpy (numpy in the same process breaks the
 * reference's iostream/locale code).
 *   okref_io fmt IN.bin            one format_g17 line per double of IN.bin
 *   okref_io vtk DIM N IN.bin OUT  write_vtk of u, w = the two halves of IN.bin
 *   okref_io cfg PATH              parse_config: the parsed values, or "ERR code: message" */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "okoracle.h"

static double* read_all(const char* path, long* n) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  const long bytes = ftell(f);
  fseek(f, 0, SEEK_SET);
  double* d = malloc((size_t)bytes + 8);
  *n = bytes / 8;
  if (fread(d, 8, (size_t)*n, f) != (size_t)*n) *n = -1;
  fclose(f);
  return d;
}

int main(int argc, char** argv) {
  long n = 0;
  if (argc == 3 && !strcmp(argv[1], "fmt")) {
    double* d = read_all(argv[2], &n);
    if (!d || n < 0) return 2;
    char buf[64];
    for (long i = 0; i < n; ++i) {
      if (oko_format_g17(d[i], buf, 64)) return 3;
      puts(buf);
    }
    return 0;
  }
  if (argc == 6 && !strcmp(argv[1], "vtk")) {
    double* d = read_all(argv[4], &n);
    if (!d || n < 0) return 2;
    if (oko_write_vtk(atoi(argv[2]), atoi(argv[3]), d, d + n / 2, argv[5])) {
      fprintf(stderr, "%s\n", oko_last_error());
      return 3;
    }
    return 0;
  }
  if (argc == 3 && !strcmp(argv[1], "cfg")) {
    static char out[1 << 16];
    const int st = oko_parse_config(argv[2], out, sizeof out);
    if (st) printf("ERR %d: %s\n", st, oko_last_error());
    else fputs(out, stdout);
    return 0;
  }
  fprintf(stderr, "usage: okref_io fmt IN.bin | okref_io vtk DIM N IN.bin OUT | okref_io cfg PATH\n");
  return 1;
}

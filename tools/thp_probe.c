// Does MADV_HUGEPAGE take effect on this host?  Maps 1 GiB, touches it and
// reports the AnonHugePages of the mapping from /proc/self/smaps.
#define _GNU_SOURCE
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
int main(void) {
  size_t sz = 1ul << 30;
  char* p = mmap(NULL, sz + (2ul << 20), PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  char* a = (char*)(((unsigned long)p + (2ul << 20) - 1) & ~((2ul << 20) - 1));
  int rc = madvise(a, sz, MADV_HUGEPAGE);
  memset(a, 1, sz);
  printf("madvise rc %d\n", rc);
  FILE* f = fopen("/proc/self/smaps", "r");
  char line[512]; int in = 0;
  while (fgets(line, sizeof line, f)) {
    unsigned long lo, hi;
    if (sscanf(line, "%lx-%lx", &lo, &hi) == 2 && strchr(line, '-') == line + strcspn(line, "-")) in = (lo <= (unsigned long)a && (unsigned long)a < hi);
    if (in && (strncmp(line, "AnonHugePages", 13) == 0 || strncmp(line, "Rss", 3) == 0 || strncmp(line, "THPeligible", 11) == 0)) fputs(line, stdout);
  }
  return 0;
}

/* First-touch cost of fresh anonymous memory on this host (the reference's compute_G
 * returns a fresh Matrix every call, factor.cpp:93): T threads touch disjoint stretches of
 * a malloc'd buffer, with and without MADV_HUGEPAGE; prints the THP policy and how much of
 * the buffer ended up on huge pages.
 *   gcc -O2 -pthread -o first_touch_probe scripts/first_touch_probe.c && ./first_touch_probe 16 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <time.h>

static double now(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec + 1e-9 * t.tv_nsec;
}
typedef struct { char* a; size_t n; } Job;
static void* touch(void* p) {
    Job* j = (Job*)p;
    for (size_t o = 0; o < j->n; o += 4096) j->a[o] = 1;
    return NULL;
}
static void show(const char* path) {
    char buf[256] = {0};
    FILE* f = fopen(path, "r");
    if (!f) { printf("%s: n/a\n", path); return; }
    if (fgets(buf, sizeof(buf), f)) printf("%s: %s", path, buf);
    fclose(f);
}
static long anon_huge_kb(void) {
    FILE* f = fopen("/proc/meminfo", "r");
    char line[256];
    long v = -1;
    while (f && fgets(line, sizeof(line), f))
        if (sscanf(line, "AnonHugePages: %ld kB", &v) == 1) break;
    if (f) fclose(f);
    return v;
}
int main(int argc, char** argv) {
    int T = argc > 1 ? atoi(argv[1]) : 16;
    size_t bytes = (size_t)(argc > 2 ? atof(argv[2]) : 8.0) * (1ull << 30);
    show("/sys/kernel/mm/transparent_hugepage/enabled");
    show("/sys/kernel/mm/transparent_hugepage/defrag");
    for (int huge = 0; huge < 2; ++huge) {
        char* a = malloc(bytes);
        if (huge) {
            uintptr_t s = ((uintptr_t)a + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
            madvise((void*)s, bytes - (s - (uintptr_t)a) - (2u << 20), MADV_HUGEPAGE);
        }
        long h0 = anon_huge_kb();
        pthread_t th[256];
        Job jobs[256];
        double t0 = now();
        for (int i = 0; i < T; ++i) {
            size_t b = bytes * i / T, e = bytes * (i + 1) / T;
            jobs[i].a = a + b;
            jobs[i].n = e - b;
            pthread_create(&th[i], NULL, touch, &jobs[i]);
        }
        for (int i = 0; i < T; ++i) pthread_join(th[i], NULL);
        double dt = now() - t0;
        long h1 = anon_huge_kb();
        printf("{\"madv_hugepage\": %d, \"threads\": %d, \"GB\": %.1f, \"seconds\": %.3f, \"GB_per_s\": %.1f, \"huge_MB\": %ld}\n",
               huge, T, bytes / 1e9, dt, bytes / dt / 1e9, (h1 - h0) / 1024);
        free(a);
    }
    return 0;
}

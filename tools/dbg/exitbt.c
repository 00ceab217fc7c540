// LD_PRELOAD helper: print a backtrace when the process calls exit/_exit
#define _GNU_SOURCE
#include <dlfcn.h>
#include <execinfo.h>
#include <stdio.h>
#include <stdlib.h>
#include <unistd.h>
static void bt(const char* who, int code) {
  void* b[64];
  int n = backtrace(b, 64);
  fprintf(stderr, "== %s(%d) called from:\n", who, code);
  backtrace_symbols_fd(b, n, 2);
}
void exit(int code) {
  bt("exit", code);
  void (*real)(int) = (void (*)(int))dlsym(RTLD_NEXT, "exit");
  real(code);
  for (;;) {}
}
void _exit(int code) {
  bt("_exit", code);
  void (*real)(int) = (void (*)(int))dlsym(RTLD_NEXT, "_exit");
  real(code);
  for (;;) {}
}

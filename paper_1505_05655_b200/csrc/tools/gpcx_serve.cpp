// gpcx_serve.cpp -- `gpcx-serve`: the B200 task server as a process, the
// counterpart of the reference CLI's `gpc serve` (proj/tools/gpc.cpp:94-128):
// same flags where they apply (--bind, --port, --max-tasks, --timeout /
// --timeout-secs), the
// same shutdown (SIGINT / SIGTERM blocked before the server threads exist,
// consumed by sigwait, then a draining stop) and a one-line banner.  The
// registry it serves is libgpcx's: LUT_GEN / LUT_APPLY / LUT_CORRECT /
// MATMUL plus the reference's BAYER_* / LSQ_POLYFIT / DEVINFO, all on the
// GPUs bound with --devices (default: every visible device).
//
//   gpcx-serve [--bind 0.0.0.0] [--port 5555] [--max-tasks N] [--timeout S]
//              [--max-pending N] [--devices 0,1,...]
//
// Talks only to the C ABI (include/gpcx.h).
#include <pthread.h>
#include <signal.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../../include/gpcx.h"

namespace {

constexpr int kExitOk = 0, kExitUsage = 2, kExitFailed = 1;

void usage(const char* argv0) {
  std::fprintf(stderr,
               "usage: %s [--bind ADDR] [--port N] [--max-tasks N] [--timeout SECONDS]\n"
               "          [--max-pending N] [--devices 0,1,...]\n",
               argv0);
}

bool parse_int(const char* s, long lo, long hi, long* out) {
  char* end = nullptr;
  const long v = std::strtol(s, &end, 10);
  if (end == s || *end != '\0' || v < lo || v > hi) return false;
  *out = v;
  return true;
}

}  // namespace

int main(int argc, char** argv) {
  std::string bind = "0.0.0.0";
  long port = 5555, max_tasks = 0, timeout_secs = 30;
  std::vector<int> devices;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    const char* v = i + 1 < argc ? argv[i + 1] : nullptr;
    if (a == "-h" || a == "--help") {
      usage(argv[0]);
      return kExitOk;
    }
    if (v == nullptr) {
      usage(argv[0]);
      return kExitUsage;
    }
    long n = 0;
    if (a == "--bind") {
      bind = v;
    } else if (a == "--port" && parse_int(v, 0, 65535, &n)) {
      port = n;
    } else if (a == "--max-tasks" && parse_int(v, 0, 4096, &n)) {
      max_tasks = n;
    } else if ((a == "--timeout" || a == "--timeout-secs") && parse_int(v, 1, 86400, &n)) {
      timeout_secs = n;
    } else if (a == "--max-pending" && parse_int(v, 1, 1 << 20, &n)) {
      // admission control of the staged server (include/gpcx.h): read from
      // the environment when the server starts
      setenv("GPCX_MAX_PENDING", v, 1);
    } else if (a == "--devices") {
      for (const char* p = v; *p != '\0';) {
        char* end = nullptr;
        const long d = std::strtol(p, &end, 10);
        if (end == p || d < 0) {
          usage(argv[0]);
          return kExitUsage;
        }
        devices.push_back(static_cast<int>(d));
        p = *end == ',' ? end + 1 : end;
        if (*end != ',' && *end != '\0') {
          usage(argv[0]);
          return kExitUsage;
        }
      }
    } else {
      usage(argv[0]);
      return kExitUsage;
    }
    ++i;
  }

  if (gpcx_init(static_cast<int>(devices.size()), devices.empty() ? nullptr : devices.data()) != 0) {
    std::fprintf(stderr, "gpcx-serve: %s\n", gpcx_last_error());
    return kExitFailed;
  }
  int ndev = 0;
  gpcx_device_count(&ndev);

  // Block the shutdown signals before the server threads exist so they
  // inherit the mask and sigwait below is the only consumer.
  sigset_t signals;
  sigemptyset(&signals);
  sigaddset(&signals, SIGINT);
  sigaddset(&signals, SIGTERM);
  pthread_sigmask(SIG_BLOCK, &signals, nullptr);

  void* server = nullptr;
  uint16_t bound = 0;
  if (gpcx_server_start(bind.c_str(), static_cast<uint16_t>(port), static_cast<int>(max_tasks),
                        static_cast<int>(timeout_secs * 1000), &server, &bound) != 0) {
    std::fprintf(stderr, "gpcx-serve: %s\n", gpcx_last_error());
    return kExitFailed;
  }
  std::printf("gpcx server listening on %s:%u (devices=%d, max_tasks=%ld, timeout=%lds)\n",
              bind.c_str(), static_cast<unsigned>(bound), ndev, max_tasks, timeout_secs);
  std::fflush(stdout);

  int sig = 0;
  sigwait(&signals, &sig);
  std::fprintf(stderr, "signal %d, draining\n", sig);
  gpcx_server_stats st{};
  if (gpcx_server_stats_get(server, &st) == 0)
    std::fprintf(stderr, "served %llu requests (busy %llu, dropped %llu)\n",
                 static_cast<unsigned long long>(st.requests), static_cast<unsigned long long>(st.busy),
                 static_cast<unsigned long long>(st.dropped));
  const int rc = gpcx_server_stop(server);
  gpcx_shutdown();
  return rc == 0 ? kExitOk : kExitFailed;
}

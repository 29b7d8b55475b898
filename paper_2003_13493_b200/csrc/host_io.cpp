// Configuration parsing, validation and PGM I/O for the C ABI.
//
// Behaviour follows the reference exactly where the C ABI can observe it:
// key set and value syntax (config.cpp:70-131: std::stoi / std::stod with a
// whole-token check, unknown key -> ConfigError), file syntax (blank and '#'
// lines skipped, "key = value" with trimming, errors prefixed path:line),
// range checks at detector creation (fast.cpp:18-27, nms.cpp:13-23,
// lk.cpp:36-46, frontend.cpp:26-36) and the binary-PGM reader
// (image.cpp:86-170).
#include <cuda_runtime.h>

#include <cctype>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <mutex>
#include <new>
#include <unordered_set>

#include "common.hpp"

namespace flkb {

namespace {

std::string strip(const std::string& s) {
  const char* ws = " \t\r\n";
  const auto a = s.find_first_not_of(ws);
  if (a == std::string::npos) return std::string();
  return s.substr(a, s.find_last_not_of(ws) - a + 1);
}

int to_int(const std::string& key, const std::string& text) {
  size_t used = 0;
  int v = 0;
  try {
    v = std::stoi(text, &used);
  } catch (const std::exception&) {
    used = std::string::npos;
  }
  if (used != text.size()) throw ConfigError("invalid integer for '" + key + "': '" + text + "'");
  return v;
}

double to_double(const std::string& key, const std::string& text) {
  size_t used = 0;
  double v = 0.0;
  try {
    v = std::stod(text, &used);
  } catch (const std::exception&) {
    used = std::string::npos;
  }
  if (used != text.size()) throw ConfigError("invalid number for '" + key + "': '" + text + "'");
  return v;
}

}  // namespace

void validate(const Config& c) {
  if (c.epsilon < 0 || c.epsilon > 255)
    throw InvalidArgument("epsilon must be in [0, 255], got " + std::to_string(c.epsilon));
  if (c.arc_length < 9 || c.arc_length > 16)
    throw InvalidArgument("arc length must be in [9, 16], got " + std::to_string(c.arc_length));
  if (c.cell_width_units < 1 || c.cell_height_units < 1)
    throw InvalidArgument("grid cell units must be positive");
  if (c.num_levels < 1) throw InvalidArgument("grid needs at least one level");
  if (c.nms_radius < 1) throw InvalidArgument("suppression radius must be at least 1");
  if (c.max_iterations < 1) throw InvalidArgument("tracker needs at least one iteration per level");
  if (!(c.convergence_epsilon > 0.0)) throw InvalidArgument("convergence epsilon must be positive");
  if (c.target_count < 1) throw ConfigError("target track count must be positive");
  if (!(c.redetect_ratio > 0.0 && c.redetect_ratio < 1.0))
    throw ConfigError("re-detection ratio must lie strictly between 0 and 1");
  if (c.cell_width_px < 0 || c.cell_height_px < 0)
    throw InvalidArgument("cell size override must be non-negative");
  if (c.num_levels > 16) throw InvalidArgument("at most 16 pyramid levels are supported");
}

void apply_config_entry(Config* c, const std::string& key, const std::string& value) {
  if (key == "epsilon") {
    c->epsilon = to_int(key, value);
  } else if (key == "N") {
    c->arc_length = to_int(key, value);
  } else if (key == "score_kind") {
    if (value == "sad_b") c->score = ScoreKind::kSadB;
    else if (value == "sad_a") c->score = ScoreKind::kSadA;
    else if (value == "mt") c->score = ScoreKind::kMt;
    else throw ConfigError("unknown score_kind '" + value + "' (expected sad_b, sad_a, or mt)");
  } else if (key == "l") {
    c->num_levels = to_int(key, value);
  } else if (key == "w") {
    c->cell_width_units = to_int(key, value);
  } else if (key == "h") {
    c->cell_height_units = to_int(key, value);
  } else if (key == "n") {
    c->nms_radius = to_int(key, value);
  } else if (key == "target_count") {
    c->target_count = to_int(key, value);
  } else if (key == "redetect_ratio") {
    c->redetect_ratio = to_double(key, value);
  } else if (key == "param_mode") {
    if (value == "translation") c->mode = ParamMode::kTranslation;
    else if (value == "translation_offset") c->mode = ParamMode::kTranslationOffset;
    else if (value == "translation_gain") c->mode = ParamMode::kTranslationGain;
    else if (value == "full") c->mode = ParamMode::kFull;
    else throw ConfigError("unknown param_mode '" + value + "'");
  } else if (key == "max_iterations") {
    c->max_iterations = to_int(key, value);
  } else if (key == "convergence_epsilon") {
    c->convergence_epsilon = to_double(key, value);
  } else if (key == "threads") {
    c->threads = to_int(key, value);
  } else {
    throw ConfigError("unknown configuration key '" + key + "'");
  }
}

void load_config_file(Config* c, const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError(path + ": cannot open configuration file");
  std::string line;
  for (int no = 1; std::getline(in, line); ++no) {
    const std::string s = strip(line);
    if (s.empty() || s[0] == '#') continue;
    const auto eq = s.find('=');
    const std::string where = path + ":" + std::to_string(no) + ": ";
    if (eq == std::string::npos) throw ConfigError(where + "expected 'key = value'");
    const std::string key = strip(s.substr(0, eq));
    const std::string value = strip(s.substr(eq + 1));
    if (key.empty() || value.empty()) throw ConfigError(where + "expected 'key = value'");
    try {
      apply_config_entry(c, key, value);
    } catch (const ConfigError& e) {
      throw ConfigError(where + e.what());
    }
  }
}

// ------------------------------------------------------------ pinned pool

namespace {

struct PinnedPool {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;  // size -> cached pinned block
  std::unordered_set<const void*> pinned;    // every live or cached pinned block
  size_t cached = 0;
  int state = 0;  // 0 untried, 1 pinning works, -1 unavailable
  static constexpr size_t kMaxCached = size_t(256) << 20;
  static constexpr size_t kMaxPinned = size_t(8) << 30;
  size_t live_pinned = 0;
};

PinnedPool& pool() {
  static PinnedPool* p = new PinnedPool();  // never destroyed: blocks outlive static teardown
  return *p;
}

}  // namespace

void* pinned_acquire(size_t bytes) {
  if (bytes == 0) bytes = 1;
  PinnedPool& P = pool();
  {
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.free_blocks.find(bytes);
    if (it != P.free_blocks.end()) {
      void* p = it->second;
      P.free_blocks.erase(it);
      P.cached -= bytes;
      return p;
    }
    if (P.state >= 0 && P.live_pinned + bytes <= PinnedPool::kMaxPinned) {
      void* p = nullptr;
      if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) == cudaSuccess) {
        P.state = 1;
        P.pinned.insert(p);
        P.live_pinned += bytes;
        return p;
      }
      cudaGetLastError();  // clear the failed call
      if (P.state == 0) P.state = -1;  // no usable driver / device: stop trying
    }
  }
  void* p = std::malloc(bytes);
  if (!p) throw std::bad_alloc();
  return p;
}

void pinned_release(void* p, size_t bytes) noexcept {
  if (!p) return;
  if (bytes == 0) bytes = 1;
  PinnedPool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  if (P.pinned.count(p) == 0) {
    std::free(p);
    return;
  }
  if (P.cached + bytes <= PinnedPool::kMaxCached) {
    P.free_blocks.emplace(bytes, p);
    P.cached += bytes;
    return;
  }
  P.pinned.erase(p);
  P.live_pinned -= bytes;
  cudaFreeHost(p);
}

bool pinned_contains(const void* p) {
  PinnedPool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  return P.pinned.count(p) != 0;
}

HostImage make_image(int width, int height, const uint8_t* pixels) {
  if (width < 1 || height < 1)
    throw InvalidArgument("image dimensions must be positive, got " + std::to_string(width) +
                          "x" + std::to_string(height));
  HostImage img;
  img.width = width;
  img.height = height;
  img.px.assign(pixels, pixels + static_cast<size_t>(width) * height);
  return img;
}

namespace {

// One header token; '#' starts a comment to end of line. Consumes the single
// whitespace byte that terminates the token (image.cpp:96-113).
bool pgm_token(std::istream& in, std::string* tok) {
  tok->clear();
  int c = in.get();
  while (c != EOF) {
    if (c == '#') {
      while (c != EOF && c != '\n') c = in.get();
    } else if (std::isspace(c)) {
      c = in.get();
    } else {
      break;
    }
  }
  while (c != EOF && !std::isspace(c)) {
    tok->push_back(static_cast<char>(c));
    c = in.get();
  }
  return !tok->empty();
}

int pgm_int(std::istream& in, const std::string& path, const char* what) {
  std::string tok;
  if (!pgm_token(in, &tok)) throw IoError(path + ": truncated PGM header (missing " + what + ")");
  size_t used = 0;
  int v = 0;
  try {
    v = std::stoi(tok, &used);
  } catch (const std::exception&) {
    used = std::string::npos;
  }
  if (used != tok.size()) throw IoError(path + ": invalid PGM " + what + " '" + tok + "'");
  return v;
}

}  // namespace

HostImage load_pgm(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError(path + ": cannot open file");
  std::string magic;
  if (!pgm_token(in, &magic) || magic != "P5") throw IoError(path + ": not a binary PGM (P5) file");
  const int w = pgm_int(in, path, "width");
  const int h = pgm_int(in, path, "height");
  const int maxval = pgm_int(in, path, "maxval");
  if (w < 1 || h < 1) throw IoError(path + ": invalid PGM dimensions");
  if (maxval != 255)
    throw IoError(path + ": unsupported PGM maxval " + std::to_string(maxval) + " (must be 255)");
  HostImage img;
  img.width = w;
  img.height = h;
  img.px.resize(static_cast<size_t>(w) * h);
  in.read(reinterpret_cast<char*>(img.px.data()), static_cast<std::streamsize>(img.px.size()));
  if (in.gcount() != static_cast<std::streamsize>(img.px.size()))
    throw IoError(path + ": truncated PGM pixel data");
  return img;
}

void save_pgm(const HostImage& img, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError(path + ": cannot open file for writing");
  char hdr[64];
  const int n = std::snprintf(hdr, sizeof(hdr), "P5\n%d %d\n255\n", img.width, img.height);
  out.write(hdr, n);
  out.write(reinterpret_cast<const char*>(img.px.data()),
            static_cast<std::streamsize>(img.px.size()));
  if (!out) throw IoError(path + ": write failed");
}

}  // namespace flkb

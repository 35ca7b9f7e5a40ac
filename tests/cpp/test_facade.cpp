// C++ facade tests: the reference's own unit tests (proj/tests/*.cpp),
// restated against the encrypted B200 path through include/hegpu.hpp.
// Built and run by tests/test_cpp_facade.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hegpu.hpp"

using namespace hegpu;

static int failures = 0;
#define CHECK(cond)                                                  \
  do {                                                               \
    if (!(cond)) {                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
      ++failures;                                                    \
    }                                                                \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                     \
  do {                                                               \
    bool caught = false;                                             \
    try { expr; } catch (const T&) { caught = true; } catch (...) {} \
    CHECK(caught);                                                   \
  } while (0)

static bool close(double a, double b, double tol = 1e-6) { return std::fabs(a - b) <= tol; }

int main() {
  Context ctx(10, {60, 40, 40, 40}, 60, /*seed=*/99);
  const int S = ctx.slots();
  const int L = ctx.levels();
  ctx.gen_rotation_keys({1, S - 1, 2, 169, 338});
  ctx.gen_relin_key();

  // test_slotvec.cpp:34-51 rotate_right basics (slot j <- v[(j - r) mod S])
  {
    std::vector<double> v(S);
    for (int j = 0; j < S; ++j) v[j] = (j % 7) * 0.125;
    Ciphertext ct = encrypt(v, L, 1, ctx);
    ctx.reset_meter();
    Ciphertext r0 = rotate_right(ct, 0, ctx);
    CHECK(ctx.tally().rot == 0);
    Ciphertext r1 = rotate_right(ct, 1, ctx);
    CHECK(ctx.tally().rot == 1);
    const std::vector<double> d = r1.decrypt();
    bool ok = true;
    for (int j = 0; j < S; ++j) ok = ok && close(d[j], v[(j - 1 + S) % S]);
    CHECK(ok);
    CHECK_THROWS_AS(rotate_right(ct, S, ctx), std::out_of_range);
    CHECK_THROWS_AS(rotate_right(ct, -1, ctx), std::out_of_range);
    // test_slotvec.cpp:53-64 rotate_left
    Ciphertext l1 = rotate_left(ct, 1, ctx);
    const std::vector<double> e = l1.decrypt();
    CHECK(close(e[0], v[1]) && close(e[S - 1], v[0]));
    CHECK(ctx.tally().rot == 2);
    // composition: right(1) then left(1) is the identity
    const std::vector<double> id = rotate_left(r1, 1, ctx).decrypt();
    bool ok2 = true;
    for (int j = 0; j < S; ++j) ok2 = ok2 && close(id[j], v[j]);
    CHECK(ok2);
  }

  // test_slotvec.cpp:92-134 add / mul metering and values
  {
    ctx.reset_meter();
    Ciphertext a = encrypt({1, 2}, L, 2, ctx);
    Ciphertext b = encrypt({3, 4}, L, 3, ctx);
    const std::vector<double> s = add(a, b, ctx).decrypt();
    CHECK(close(s[0], 4) && close(s[1], 6));
    CHECK(ctx.tally().add_cc == 1);
    Plaintext zero(ctx, {}, a.scale(), L);
    const std::vector<double> s2 = add(a, zero, ctx).decrypt();
    CHECK(close(s2[0], 1) && close(s2[1], 2));
    CHECK(ctx.tally().add_pc == 1);
    Plaintext ones(ctx, std::vector<double>(S, 1.0), 1099511627776.0, L);
    Ciphertext p = mul(a, ones, ctx);
    CHECK(ctx.tally().mul_pc == 1);
    const std::vector<double> pr = rescale(p, ctx).decrypt();
    CHECK(close(pr[0], 1) && close(pr[1], 2));
    // square_layer (convlower.cpp:141-143): one Mul CC
    const std::vector<double> sq = square_layer(encrypt({2, -3, 0, 1}, L, 4, ctx), ctx).decrypt();
    CHECK(close(sq[0], 4) && close(sq[1], 9) && close(sq[2], 0) && close(sq[3], 1));
    CHECK(ctx.tally().mul_cc == 1);
  }

  // test_convlower.cpp:171-211 merge_maps: 3 maps of 169 slots -> 2 rot, 2 add
  {
    std::vector<uint64_t> wire;
    std::vector<std::vector<double>> vals(3, std::vector<double>(169));
    for (int j = 0; j < 3; ++j) {
      for (int p = 0; p < 169; ++p) vals[j][p] = 0.01 * ((p * (j + 3)) % 17);
      Ciphertext c = encrypt(vals[j], L, 10 + j, ctx);
      const std::vector<uint64_t> w = c.download();
      wire.insert(wire.end(), w.begin(), w.end());
    }
    Ciphertext maps(ctx, 3, L);
    maps.upload(wire, 1099511627776.0);
    ctx.reset_meter();
    const std::vector<double> m = merge_maps(maps, 3, 169, ctx).decrypt();
    CHECK(ctx.tally().rot == 2 && ctx.tally().add_cc == 2);
    bool ok = true;
    for (int j = 0; j < 3; ++j)
      for (int p = 0; p < 169; ++p) ok = ok && close(m[j * 169 + p], vals[j][p]);
    CHECK(ok);
    CHECK_THROWS_AS(merge_maps(maps, 3, S, ctx), CapacityError);
  }

  // test_matvec.cpp:88-97 HS 2x2 worked example: [[1,2],[3,4]] [5,6] = [17, 39]
  {
    HsPlan plan({1, 2, 3, 4}, 2, 2, L, ctx);
    ctx.gen_rotation_keys(plan.rotations());
    ctx.reset_meter();
    const std::vector<double> r = hs_matvec(plan, encrypt({5, 6}, L, 20, ctx), ctx).decrypt();
    CHECK(close(r[0], 17, 1e-5) && close(r[1], 39, 1e-5));
    CHECK(ctx.tally().mul_pc == 2);
  }

  // test_matvec.cpp:99-108 identity 4x4: zero diagonals skipped, one fold
  {
    std::vector<double> I(16, 0.0);
    for (int i = 0; i < 4; ++i) I[i * 4 + i] = 1.0;
    HsPlan plan(I, 4, 4, L, ctx);
    ctx.gen_rotation_keys(plan.rotations());
    ctx.reset_meter();
    const std::vector<double> x = {0.25, -0.5, 0.75, 0.125};
    const std::vector<double> r = hs_matvec(plan, encrypt(x, L, 21, ctx), ctx).decrypt();
    for (int i = 0; i < 4; ++i) CHECK(close(r[i], x[i], 1e-5));
    CHECK(ctx.tally().mul_pc == 1);
    CHECK(ctx.tally().rot == 1);
  }

  // test_matvec.cpp:298-304 capacity violations throw
  CHECK_THROWS_AS(HsPlan(std::vector<double>(4 * (S + 1), 1.0), 4, S + 1, L, ctx), CapacityError);

  // test_netcompile.cpp "model json round trip and validation" (modelio)
  {
    const ModelSpec m = parse_model_json(R"({"name": "tiny", "input": [1, 4, 4], "n_slots": 32, "layers": [
      {"kind": "conv", "k": 3, "s": 1, "out_channels": 2, "label": "Conv1"}, {"kind": "square"},
      {"kind": "flatten"}, {"kind": "dense", "units": 3, "label": "Dense1"}]})");
    CHECK(m.weight_floats() == 2 * 9 + 2 + 3 * 8 + 3);
    CHECK_THROWS_AS(parse_model_json(R"({"name":"x"})"), IoError);
    CHECK_THROWS_AS(parse_model_json(R"({"name":"x","input":[1,2,2],"n_slots":8,"layers":[],"extra":1})"), IoError);
    CHECK_THROWS_AS(parse_model_json(R"({"name":"x","input":[1,2,2],"n_slots":8,
                                         "layers":[{"kind":"dense","units":1,"typo_field":2}]})"),
                    IoError);
    CHECK_THROWS_AS(load_weights(m, "/nonexistent/w.bin"), IoError);
  }

  // test_netcompile.cpp:40-54 lower(): stage labels; :74-97 a single 1x1 dense
  // model costs one multiplication and no rotation; execute() through the
  // general stage driver (grouped SubConv stages + the conv-pack repack)
  {
    const ModelSpec unit = parse_model_json(R"({"name": "unit", "input": [1, 1, 1], "n_slots": 512, "layers": [
      {"kind": "dense", "units": 1, "label": "D"}]})");
    const std::vector<Stage> st = lower(unit);
    CHECK(st.size() == 1 && st[0].kind == StageKind::Linear && st[0].label == "D");
    Context c2(10, {45, 40}, 45, /*seed=*/5);
    LoweredProgram prog(c2, unit, {3.0, 1.0});
    const ExecResult r = execute(prog, {2.0}, 1);
    CHECK(close(r.logits[0], 7.0, 1e-5));
    CHECK(r.report.total.mul_pc == 1);
    CHECK(r.report.total.rot == 0);

    const ModelSpec grouped = parse_model_json(R"({"name": "g", "input": [2, 6, 6], "n_slots": 512, "layers": [
      {"kind": "conv", "k": 3, "s": 1, "out_channels": 4, "label": "Conv1"}, {"kind": "square"},
      {"kind": "subconv", "k": 2, "s": 1, "out_channels": 4, "groups": 2, "label": "Conv2"},
      {"kind": "conv", "k": 1, "s": 1, "out_channels": 3, "policy": "convpack", "label": "Conv3"},
      {"kind": "square"}, {"kind": "flatten"}, {"kind": "dense", "units": 2, "label": "Dense1"}]})");
    const std::vector<Stage> gs = lower(grouped);
    const char* want[] = {"Conv1", "Flat1", "Square1", "Conv2", "Conv3", "Flat2", "Square2", "Dense1"};
    CHECK(gs.size() == 8);
    for (size_t i = 0; i < gs.size() && i < 8; ++i) CHECK(gs[i].label == want[i]);
    CHECK(gs.size() == 8 && gs[1].groups == 2 && gs[3].groups == 2 && gs[4].kind == StageKind::RepackConv);
    // zero weights give all-zero logits (test_netcompile.cpp:154-171)
    Context c3(10, {45, 40, 40, 40, 40, 40, 40}, 45, /*seed=*/6);
    LoweredProgram zp(c3, grouped, std::vector<double>(grouped.weight_floats(), 0.0));
    std::vector<double> img(2 * 6 * 6);
    for (size_t i = 0; i < img.size(); ++i) img[i] = 0.01 * (double)(i % 17);
    const ExecResult z = execute(zp, img, 3);
    CHECK(z.logits.size() == 2 && close(z.logits[0], 0.0, 1e-5) && close(z.logits[1], 0.0, 1e-5));
    CHECK(z.report.rows.size() == 8 && z.report.rows[4].first == "Conv3");
    // a LoLa-stacked stage policy is a ShapeError; a short chain a CapacityError
    const ModelSpec stacked = parse_model_json(R"({"name": "s", "input": [1, 2, 2], "n_slots": 512, "layers": [
      {"kind": "flatten"}, {"kind": "dense", "units": 2, "policy": "lola-stacked", "label": "D1"}]})");
    CHECK_THROWS_AS(LoweredProgram(c2, stacked, std::vector<double>(stacked.weight_floats(), 0.0)), ShapeError);
    CHECK_THROWS_AS(LoweredProgram(c2, grouped, std::vector<double>(grouped.weight_floats(), 0.0)), CapacityError);
  }

  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}

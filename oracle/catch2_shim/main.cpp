// Runner for the Catch2 shim: prints one line per test case and a JSON summary.
#include <catch2/catch_amalgamated.hpp>
#include <cstring>

int main(int argc, char** argv) {
    int failed = 0, passed = 0;
    for (const auto& c : catch_shim::registry()) {
        if (argc > 1 && std::strstr(c.name, argv[1]) == nullptr) continue;
        try {
            c.fn();
            ++passed;
            std::printf("PASS  %s\n", c.name);
        } catch (const catch_shim::Failure& f) {
            ++failed;
            std::printf("FAIL  %s  (%s)\n", c.name, f.what.c_str());
        } catch (const std::exception& e) {
            ++failed;
            std::printf("FAIL  %s  (uncaught exception: %s)\n", c.name, e.what());
        }
    }
    std::printf("{\"cases_passed\": %d, \"cases_failed\": %d, \"checks\": %ld}\n", passed, failed,
                catch_shim::checks());
    return failed == 0 ? 0 : 1;
}
